python scripts/host_tier_gather.py > gpurun_out/r2n_host_gather.txt 2>&1
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/r2n_bench20.json 2> gpurun_out/r2n_bench20.err
