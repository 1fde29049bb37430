timeout 1500 python -m pytest tests -m gpu -q -x --durations=10 2>&1 | tail -40 > gpurun_out/r2c_tests.txt
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/r2c_bench.json 2> gpurun_out/r2c_bench.err
timeout 600 python bench.py --steps 200 --warmup 20 --no-cpu-baseline > gpurun_out/r2c_bench200.json 2> gpurun_out/r2c_bench200.err
