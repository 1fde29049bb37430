python scripts/dbg/rej_debug.py > gpurun_out/r2d_rej.txt 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/r2d_launches.csv python bench.py --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/r2d_ncu_bench.log 2>&1
timeout 600 python bench.py --steps 200 --warmup 20 --no-cpu-baseline > gpurun_out/r2d_bench200.json 2> gpurun_out/r2d_bench200.err
