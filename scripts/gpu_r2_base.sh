# Round-2 baseline on a fresh box: GPU tests, smoke, default bench, papers_bm bench, launch list.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/base_gpu.txt 2>&1
lscpu > gpurun_out/base_lscpu.txt 2>&1
timeout 1500 python -m pytest tests/ -q -x -m gpu > gpurun_out/base_tests.txt 2>&1; echo "tests rc=$?" >> gpurun_out/base_tests.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/base_smoke.txt 2>&1
timeout 900 python bench.py > gpurun_out/base_bench.json 2> gpurun_out/base_bench.err
timeout 900 python bench.py --config papers_bm --steps 20 --warmup 5 > gpurun_out/base_bench_bm.json 2> gpurun_out/base_bench_bm.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -s 400 -c 400 --csv --log-file gpurun_out/base_launches.csv \
    python bench.py --steps 60 --warmup 5 --no-cpu-baseline --no-per-call > gpurun_out/base_launches_bench.log 2>&1
