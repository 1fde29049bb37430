timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/r2j_bench20.json 2> gpurun_out/r2j_bench20.err
timeout 600 python bench.py --config products --steps 20 --warmup 5 --no-cpu-baseline --no-per-call > gpurun_out/r2j_products.json 2> gpurun_out/r2j_products.err
timeout 900 python bench.py --config papers_host_bm --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/r2j_hostbm.json 2> gpurun_out/r2j_hostbm.err
timeout 600 python -m pytest tests/test_gpu_parity.py -q -m gpu -k "pipeline" 2>&1 | tail -3 > gpurun_out/r2j_tests.txt
