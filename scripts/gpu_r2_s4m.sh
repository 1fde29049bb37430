# Functional check of the multi-rank bench path on a 1-GPU box (two ranks share the GPU).
mkdir -p gpurun_out
timeout 1200 python bench.py --gpus 2 --steps 40 --warmup 5 --no-cpu-baseline --no-per-call > gpurun_out/s4m_bench_gpus2.json 2> gpurun_out/s4m_bench_gpus2.err; echo "rc=$?" >> gpurun_out/s4m_bench_gpus2.err
timeout 900 python bench.py --impl reference --gpus 2 --steps 8 --warmup 1 > gpurun_out/s4m_ref_gpus2.json 2> gpurun_out/s4m_ref_gpus2.err; echo "rc=$?" >> gpurun_out/s4m_ref_gpus2.err
