# Host enqueue cost per batch vs the device step (is the runner host-bound?).
mkdir -p gpurun_out
K=300 timeout 600 python scripts/ab.py "S=8" "S=8,cs=1" > gpurun_out/s3m_ab.txt 2>&1
K=200 timeout 600 python scripts/ab.py "S=8,bm=11105995" >> gpurun_out/s3m_ab.txt 2>&1
