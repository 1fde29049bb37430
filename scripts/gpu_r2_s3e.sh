# Hash probing A/B: base (per-entry probes), new2 (home CAS, then 4-entry groups for inserts and
# lookups), lk (4-entry group lookups only).
mkdir -p gpurun_out
for cfg in papers products; do
  for rep in 1 2; do
    for v in base new2 lk; do
      export FDG_DBG_LIB=variants/libfdg_$v.so
      echo "== $cfg $v rep $rep" >> gpurun_out/s3e_ab.txt
      CFG=$cfg K=300 timeout 600 python scripts/ab.py "S=8" "S=8,mode=sample" 2>&1 | grep us/batch >> gpurun_out/s3e_ab.txt
    done
  done
done
