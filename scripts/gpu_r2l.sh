python scripts/startup_trace.py > gpurun_out/r2l_startup.txt 2>&1
python scripts/startup_trace.py prefetch_upfront=1 > gpurun_out/r2l_startup_upfront.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -5 > gpurun_out/r2l_tests.txt
