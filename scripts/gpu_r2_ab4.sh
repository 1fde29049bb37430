mkdir -p gpurun_out
K=300 timeout 900 python scripts/ab.py "S=8" "S=8,gather_evict_first=1" "S=8,gather_evict_first=2" "S=8,gather_evict_first=3" "S=4,gather_evict_first=1" "S=6,gather_evict_first=1" "S=8,hash_keep=0" "S=8,hash_load_pct=70" > gpurun_out/ab4.txt 2>&1
