# Buffer manager persistent grids (select / compaction) at 1 / 2 (default) / 4 CTAs per SM.
mkdir -p gpurun_out
FDG_DBG_LIB=variants/libfdg_bmp4.so timeout 1200 python -m pytest tests/test_gpu_scale.py tests/test_gpu_parity.py -q -x -k "scale or buffer_manager" > gpurun_out/s4y_tests.txt 2>&1; echo "rc=$?" >> gpurun_out/s4y_tests.txt
for rep in 1 2; do
  for v in new bmp1 bmp4; do
    if [ $v = new ]; then unset FDG_DBG_LIB; else export FDG_DBG_LIB=variants/libfdg_$v.so; fi
    echo "== $v rep $rep" >> gpurun_out/s4y_ab.txt
    K=200 timeout 900 python scripts/ab.py "S=8,bm=11105995" "S=8,bm=11105995,cs=1" 2>&1 | grep us/batch >> gpurun_out/s4y_ab.txt
  done
done
