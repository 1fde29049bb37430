# Group-probed batch hash (4 entries per L2 round trip) vs the per-entry probe (base), and the
# expansion at 40 registers (minb6). Papers then products; GPU tests first.
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_sage.py -q -x > gpurun_out/s3d_tests.txt 2>&1; echo "rc=$?" >> gpurun_out/s3d_tests.txt
for cfg in papers products; do
  for rep in 1 2; do
    for v in base new minb6; do
      if [ $v = new ]; then unset FDG_DBG_LIB; else export FDG_DBG_LIB=variants/libfdg_$v.so; fi
      echo "== $cfg $v rep $rep" >> gpurun_out/s3d_ab.txt
      CFG=$cfg K=300 timeout 600 python scripts/ab.py "S=8" "S=8,mode=sample" "S=8,cs=1" 2>&1 | grep us/batch >> gpurun_out/s3d_ab.txt
    done
  done
done
unset FDG_DBG_LIB
