# Round-2 final measurement pass: GPU tests, smoke, every config's bench line, the reference arm,
# the launch list of the default bench, whole-step DRAM traffic (Papers, config 3).
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/fin_gpu.txt 2>&1
timeout 1800 python -m pytest tests/ -q -x -m gpu > gpurun_out/fin_tests.txt 2>&1; echo "tests rc=$?" >> gpurun_out/fin_tests.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/fin_smoke.txt 2>&1
timeout 900 python bench.py > gpurun_out/fin_bench_papers.json 2> gpurun_out/fin_bench_papers.err
timeout 900 python bench.py --config papers_bm --steps 100 --warmup 20 > gpurun_out/fin_bench_papers_bm.json 2> gpurun_out/fin_bench_papers_bm.err
timeout 900 python bench.py --config products > gpurun_out/fin_bench_products.json 2> gpurun_out/fin_bench_products.err
timeout 900 python bench.py --config friendster --steps 300 > gpurun_out/fin_bench_friendster.json 2> gpurun_out/fin_bench_friendster.err
timeout 1200 python bench.py --config mag --steps 200 --warmup 10 --no-per-call > gpurun_out/fin_bench_mag.json 2> gpurun_out/fin_bench_mag.err
timeout 1200 python bench.py --config papers_host_bm --steps 20 --warmup 5 > gpurun_out/fin_bench_papers_host_bm.json 2> gpurun_out/fin_bench_papers_host_bm.err
timeout 1200 python bench.py --train --steps 200 --warmup 10 --no-per-call --no-cpu-baseline > gpurun_out/fin_bench_papers_train.json 2> gpurun_out/fin_bench_papers_train.err
timeout 900 python bench.py --impl reference --steps 64 --warmup 3 > gpurun_out/fin_reference_papers.json 2> gpurun_out/fin_reference_papers.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -s 400 -c 400 --csv --log-file gpurun_out/fin_launches.csv \
    python bench.py --steps 60 --warmup 5 --no-cpu-baseline --no-per-call > gpurun_out/fin_launches_bench.log 2>&1
FDG_PROFILE_RANGE=1 K=50 timeout 900 ncu --replay-mode app-range \
  --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --csv \
  --log-file gpurun_out/fin_range_papers.csv python scripts/ab.py S=8 > /dev/null 2>&1
FDG_PROFILE_RANGE=1 K=100 timeout 600 ncu --replay-mode app-range \
  --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --csv \
  --log-file gpurun_out/fin_range_sample.csv python scripts/ab.py "S=8,mode=sample" > /dev/null 2>&1
