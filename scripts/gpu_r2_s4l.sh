# Config-3 timeline after the buffer-manager changes.
mkdir -p gpurun_out
BM=11105995 K=200 timeout 900 python scripts/trace_pipeline.py 8 > gpurun_out/s4l_trace_bm.txt 2>&1
cp gpurun_out/trace.csv gpurun_out/s4l_trace_bm.csv 2>/dev/null
