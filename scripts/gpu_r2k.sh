python scripts/startup_trace.py > gpurun_out/r2k_startup.txt 2>&1
CFG=products python scripts/startup_trace.py > gpurun_out/r2k_startup_products.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -5 > gpurun_out/r2k_tests.txt
