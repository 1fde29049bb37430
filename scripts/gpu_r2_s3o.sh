# With 32 hardware queues: sampler count, hash load factor and L2 residency hints, re-swept.
mkdir -p gpurun_out
K=300 timeout 900 python scripts/ab.py "S=8" "S=8,hash_load_pct=70" "S=8,hash_load_pct=35" "S=8,hash_keep=0" "S=6" "S=10" "S=12" "S=8,G=2" "S=8" > gpurun_out/s3o_ab.txt 2>&1
K=300 timeout 900 python scripts/ab.py "S=8,cs=1" "S=10,cs=1" "S=12,cs=1" "S=8,cs=1,hash_load_pct=70" >> gpurun_out/s3o_ab.txt 2>&1
