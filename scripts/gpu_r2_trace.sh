# Sampler chain timelines: one sampler sample-only, eight samplers sample-only, eight samplers full.
mkdir -p gpurun_out
FLAGS=1 K=100 timeout 300 python scripts/trace_pipeline.py 1 > gpurun_out/trace_S1_sample.txt 2>&1; cp gpurun_out/trace.csv gpurun_out/trace_S1_sample.csv
FLAGS=1 K=200 timeout 300 python scripts/trace_pipeline.py 8 > gpurun_out/trace_S8_sample.txt 2>&1; cp gpurun_out/trace.csv gpurun_out/trace_S8_sample.csv
K=200 timeout 300 python scripts/trace_pipeline.py 8 > gpurun_out/trace_S8_full.txt 2>&1; cp gpurun_out/trace.csv gpurun_out/trace_S8_full.csv
