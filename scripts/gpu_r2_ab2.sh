mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -m gpu -k "sample or khop or pipeline or replay or reject" > gpurun_out/ab2_tests.txt 2>&1
K=300 timeout 900 python scripts/ab.py "S=8" "S=8,mode=sample" "S=12,mode=sample" "S=8,mode=extract" > gpurun_out/ab2.txt 2>&1
