# Sampler: early-table load factor, and the intern passes' occupancy (min-blocks builds).
mkdir -p gpurun_out
K=300 timeout 900 python scripts/ab.py "S=8" "S=8,hash_early_pct=25" "S=8,hash_early_pct=15" "S=8,mode=sample" "S=8,mode=sample,hash_early_pct=25" "S=8,cs=1" "S=8,cs=1,hash_early_pct=25" 2>&1 | grep us/batch > gpurun_out/s3q_ab.txt
for v in il6 il8 im3; do
  echo "== $v" >> gpurun_out/s3q_ab.txt
  FDG_DBG_LIB=variants/libfdg_$v.so K=300 timeout 900 python scripts/ab.py "S=8" "S=8,mode=sample" 2>&1 | grep us/batch >> gpurun_out/s3q_ab.txt
done
