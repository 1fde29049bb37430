timeout 1500 python -m pytest tests -m gpu -q -x --durations=10 2>&1 | tail -30 > gpurun_out/r2f_tests.txt
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/r2f_bench20.json 2> gpurun_out/r2f_bench20.err
timeout 600 python bench.py --steps 200 --warmup 20 --no-cpu-baseline > gpurun_out/r2f_bench200.json 2> gpurun_out/r2f_bench200.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r2f_launches.csv python bench.py --steps 20 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
