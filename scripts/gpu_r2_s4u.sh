# Next-frontier intern passes: lean at 64 registers (indptr reloaded), lean at 80 (kept), general (128); 3 reps.
mkdir -p gpurun_out
FDG_DBG_LIB=variants/libfdg_lean80.so timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "sample" > gpurun_out/s4u_tests.txt 2>&1; echo "rc=$?" >> gpurun_out/s4u_tests.txt
for rep in 1 2 3; do
  for v in new lean64 lean80; do
    if [ $v = new ]; then unset FDG_DBG_LIB; else export FDG_DBG_LIB=variants/libfdg_$v.so; fi
    echo "== $v rep $rep" >> gpurun_out/s4u_ab.txt
    K=300 timeout 900 python scripts/ab.py "S=8" "S=8,cs=1" 2>&1 | grep us/batch >> gpurun_out/s4u_ab.txt
    CFG=products K=196 timeout 900 python scripts/ab.py "S=8,cs=1" 2>&1 | grep us/batch >> gpurun_out/s4u_ab.txt
  done
done
