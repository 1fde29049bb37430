# Full GPU tests after the buffer-manager select/bind fusion; config-3 bench line.
mkdir -p gpurun_out
timeout 1800 python -m pytest tests/ -q -x -m gpu > gpurun_out/s3w_tests.txt 2>&1; echo "tests rc=$?" >> gpurun_out/s3w_tests.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/s3w_smoke.txt 2>&1
timeout 900 python bench.py --config papers_bm --steps 100 --warmup 20 > gpurun_out/s3w_bench_papers_bm.json 2> gpurun_out/s3w_bench_papers_bm.err
