# A/B of the fused gather+checksum kernels (e2e path) on the Papers and Friendster shapes
for cfg in papers friendster; do
echo "== $cfg"
CFG=$cfg timeout 300 python scripts/ab.py "S=6" "S=6,cs=1" "S=6,cs=1,hash_chunk=128" "S=6,cs=1,hash_chunk=256" "S=6,mode=extract" "S=6,mode=extract,cs=1,hash_chunk=128" "S=6,mode=extract,cs=1,hash_chunk=256"
done
