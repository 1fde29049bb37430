# Passes with a next frontier at two registers per item (intern_tile_next, 64 registers) vs the
# general tile (128 registers).
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "sample or pipeline or u64" > gpurun_out/s4j_tests.txt 2>&1; echo "rc=$?" >> gpurun_out/s4j_tests.txt
for rep in 1 2; do
  for v in nolean new; do
    if [ $v = new ]; then unset FDG_DBG_LIB; else export FDG_DBG_LIB=variants/libfdg_$v.so; fi
    echo "== $v rep $rep" >> gpurun_out/s4j_ab.txt
    K=300 timeout 900 python scripts/ab.py "S=8" "S=8,mode=sample" "S=8,cs=1" 2>&1 | grep us/batch >> gpurun_out/s4j_ab.txt
    CFG=products K=196 timeout 900 python scripts/ab.py "S=8" 2>&1 | grep us/batch >> gpurun_out/s4j_ab.txt
  done
done
