# Closing pass 4: GPU tests, smoke, Papers / products / config-3 bench lines on the final code.
mkdir -p gpurun_out
timeout 1800 python -m pytest tests/ -q -x -m gpu > gpurun_out/fin4_tests.txt 2>&1; echo "tests rc=$?" >> gpurun_out/fin4_tests.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/fin4_smoke.txt 2>&1
timeout 900 python bench.py > gpurun_out/fin4_bench_papers.json 2> gpurun_out/fin4_bench_papers.err
timeout 900 python bench.py --config products > gpurun_out/fin4_bench_products.json 2> gpurun_out/fin4_bench_products.err
timeout 900 python bench.py --config papers_bm --steps 100 --warmup 20 > gpurun_out/fin4_bench_papers_bm.json 2> gpurun_out/fin4_bench_papers_bm.err
timeout 900 python bench.py --config friendster --steps 300 > gpurun_out/fin4_bench_friendster.json 2> gpurun_out/fin4_bench_friendster.err
