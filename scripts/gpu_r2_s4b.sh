# Round-2 final measurement pass: GPU tests, smoke, every config's bench line, reference arm,
# launch list, whole-step DRAM traffic, the config-3 move's DRAM bytes.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/s4b_gpu.txt 2>&1
timeout 1800 python -m pytest tests/ -q -x -m gpu > gpurun_out/s4b_tests.txt 2>&1; echo "tests rc=$?" >> gpurun_out/s4b_tests.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/s4b_smoke.txt 2>&1
timeout 900 python bench.py > gpurun_out/s4b_bench_papers.json 2> gpurun_out/s4b_bench_papers.err
timeout 900 python bench.py --config papers_bm --steps 100 --warmup 20 > gpurun_out/s4b_bench_papers_bm.json 2> gpurun_out/s4b_bench_papers_bm.err
timeout 900 python bench.py --config products > gpurun_out/s4b_bench_products.json 2> gpurun_out/s4b_bench_products.err
timeout 900 python bench.py --config friendster --steps 300 > gpurun_out/s4b_bench_friendster.json 2> gpurun_out/s4b_bench_friendster.err
timeout 900 python bench.py --impl reference --steps 64 --warmup 3 > gpurun_out/s4b_reference_papers.json 2> gpurun_out/s4b_reference_papers.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -s 400 -c 400 --csv --log-file gpurun_out/s4b_launches.csv \
    python bench.py --steps 60 --warmup 5 --no-cpu-baseline --no-per-call > gpurun_out/s4b_launches_bench.log 2>&1
K=40 timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --cache-control none --clock-control none \
  -k regex:"k_move_hash_rb" -s 20 -c 6 --csv --log-file gpurun_out/s4b_move_traffic.csv python scripts/ab.py S=8,bm=11105995 > /dev/null 2>&1
FDG_PROFILE_RANGE=1 K=50 timeout 900 ncu --replay-mode app-range \
  --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --csv \
  --log-file gpurun_out/s4b_range_papers_bm.csv python scripts/ab.py S=8,bm=11105995 > /dev/null 2>&1
