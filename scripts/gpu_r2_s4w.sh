# Buffer-manager metadata kernels at 128 / 256 (default) / 512 threads per CTA (tile = 8 items per thread).
mkdir -p gpurun_out
for v in bmt128 bmt512; do
  FDG_DBG_LIB=variants/libfdg_$v.so timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "buffer_manager or extractor" > gpurun_out/s4w_tests_$v.txt 2>&1; echo "rc=$?" >> gpurun_out/s4w_tests_$v.txt
done
for rep in 1 2; do
  for v in new bmt128 bmt512; do
    if [ $v = new ]; then unset FDG_DBG_LIB; else export FDG_DBG_LIB=variants/libfdg_$v.so; fi
    echo "== $v rep $rep" >> gpurun_out/s4w_ab.txt
    K=200 timeout 900 python scripts/ab.py "S=8,bm=11105995" "S=8,bm=11105995,cs=1" 2>&1 | grep us/batch >> gpurun_out/s4w_ab.txt
  done
done
