# Expansion with the fanout at compile time (unrolled Floyd chain) vs runtime fanout.
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "sample" > gpurun_out/s4i_tests.txt 2>&1; echo "rc=$?" >> gpurun_out/s4i_tests.txt
for rep in 1 2; do
  for v in nofc new; do
    if [ $v = new ]; then unset FDG_DBG_LIB; else export FDG_DBG_LIB=variants/libfdg_$v.so; fi
    echo "== $v rep $rep" >> gpurun_out/s4i_ab.txt
    K=300 timeout 900 python scripts/ab.py "S=8" "S=8,mode=sample" "S=8,cs=1" 2>&1 | grep us/batch >> gpurun_out/s4i_ab.txt
    CFG=products K=196 timeout 900 python scripts/ab.py "S=8" 2>&1 | grep us/batch >> gpurun_out/s4i_ab.txt
  done
done
CFG=friendster K=200 timeout 900 python scripts/ab.py "S=8" "S=8,cs=1" 2>&1 | grep us/batch >> gpurun_out/s4i_ab.txt
FDG_DBG_LIB=variants/libfdg_nofc.so CFG=friendster K=200 timeout 900 python scripts/ab.py "S=8" "S=8,cs=1" 2>&1 | grep us/batch >> gpurun_out/s4i_ab.txt
