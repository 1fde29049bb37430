# Last-layer table load factor alone (the early table kept at 0.5), with the Bloom filter in place.
mkdir -p gpurun_out
for rep in 1 2; do
  K=300 timeout 900 python scripts/ab.py "S=8" "S=8,hash_load_pct=60,hash_early_pct=50" "S=8,hash_load_pct=40,hash_early_pct=50" "S=8,cs=1" "S=8,cs=1,hash_load_pct=60,hash_early_pct=50" 2>&1 | grep us/batch >> gpurun_out/s5f_ab.txt
done
