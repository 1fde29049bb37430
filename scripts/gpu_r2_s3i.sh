# Config-3 timeline (in-library tracer): in-situ durations of the buffer-manager kernels.
mkdir -p gpurun_out
BM=11105995 K=200 timeout 900 python scripts/trace_pipeline.py 8 > gpurun_out/s3i_trace_bm.txt 2>&1
cp gpurun_out/trace.csv gpurun_out/s3i_trace_bm.csv 2>/dev/null
BM=11105995 K=200 FLAGS=2 timeout 900 python scripts/trace_pipeline.py 8 > gpurun_out/s3i_trace_bm_extract.txt 2>&1
