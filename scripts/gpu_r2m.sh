timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -m gpu -k "mt or pipeline or lemire or sample" 2>&1 | tail -3 > gpurun_out/r2m_tests.txt
python scripts/startup_trace.py > gpurun_out/r2m_startup.txt 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_mt -c 20 --csv --log-file gpurun_out/r2m_mt.csv python scripts/startup_trace.py > /dev/null 2>&1
CFG=papers K=300 timeout 900 python scripts/ab.py "S=8" "S=8,mode=sample" >> gpurun_out/r2m_ab.txt 2>&1
