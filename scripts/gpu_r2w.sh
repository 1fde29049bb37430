timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -m gpu -k "host_tier or buffer" 2>&1 | tail -3 > gpurun_out/r2w_tests.txt
python scripts/host_tier_gather.py 111059956 0 > gpurun_out/r2w_host.txt 2>&1
timeout 900 python bench.py --config papers_host_bm --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/r2w_hostbm.json 2> gpurun_out/r2w_hostbm.err
