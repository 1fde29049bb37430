# Last check on the final code: all GPU tests, smoke, the default bench line.
mkdir -p gpurun_out
timeout 1800 python -m pytest tests/ -q -x -m gpu > gpurun_out/last_tests.txt 2>&1; echo "tests rc=$?" >> gpurun_out/last_tests.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/last_smoke.txt 2>&1
timeout 900 python bench.py > gpurun_out/last_bench_papers.json 2> gpurun_out/last_bench_papers.err
