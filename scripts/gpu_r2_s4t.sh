# e2e form (fused checksum): total CTA count of the hashing gather.
mkdir -p gpurun_out
for rep in 1 2; do
  K=300 timeout 900 python scripts/ab.py "S=8,cs=1" "S=8,cs=1,hash_ctas=74" "S=8,cs=1,hash_ctas=111" "S=8,cs=1,hash_ctas=222" 2>&1 | grep us/batch >> gpurun_out/s4t_ab.txt
done
CFG=products K=196 timeout 900 python scripts/ab.py "S=8,cs=1" "S=8,cs=1,hash_ctas=111" "S=8,cs=1,hash_ctas=222" 2>&1 | grep us/batch >> gpurun_out/s4t_ab.txt
