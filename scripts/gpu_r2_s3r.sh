# Round-2 measurement pass: GPU tests, smoke, every config's bench line, the reference arm,
# the launch list of the default bench.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/s3r_gpu.txt 2>&1
timeout 1500 python -m pytest tests/ -q -x -m gpu > gpurun_out/s3r_tests.txt 2>&1; echo "tests rc=$?" >> gpurun_out/s3r_tests.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/s3r_smoke.txt 2>&1
timeout 900 python bench.py > gpurun_out/s3r_bench_papers.json 2> gpurun_out/s3r_bench_papers.err
timeout 900 python bench.py --config papers_bm --steps 100 --warmup 20 > gpurun_out/s3r_bench_papers_bm.json 2> gpurun_out/s3r_bench_papers_bm.err
timeout 900 python bench.py --config products > gpurun_out/s3r_bench_products.json 2> gpurun_out/s3r_bench_products.err
timeout 900 python bench.py --config friendster --steps 300 > gpurun_out/s3r_bench_friendster.json 2> gpurun_out/s3r_bench_friendster.err
timeout 900 python bench.py --impl reference --steps 64 --warmup 3 > gpurun_out/s3r_reference_papers.json 2> gpurun_out/s3r_reference_papers.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -s 400 -c 400 --csv --log-file gpurun_out/s3r_launches.csv \
    python bench.py --steps 60 --warmup 5 --no-cpu-baseline --no-per-call > gpurun_out/s3r_launches_bench.log 2>&1
