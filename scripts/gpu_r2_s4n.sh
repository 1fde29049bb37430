# Products e2e form: fused checksum chunk size and CTAs per SM for 400-byte rows.
mkdir -p gpurun_out
for rep in 1 2; do
  CFG=products K=196 timeout 900 python scripts/ab.py "S=8,cs=1" "S=8,cs=1,hash_chunk=128" "S=8,cs=1,hash_chunk=128,hash_ctas_per_sm=2" "S=8,cs=1,hash_ctas_per_sm=2" "S=8" 2>&1 | grep us/batch >> gpurun_out/s4n_ab.txt
done
