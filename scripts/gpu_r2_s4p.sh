# Buffer manager without the two counter-reset launches per batch: parity + A/B.
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_scale.py tests/test_cpp_shim.py tests/test_session.py tests/test_gpu_dataset.py -q -x > gpurun_out/s4p_tests.txt 2>&1; echo "rc=$?" >> gpurun_out/s4p_tests.txt
for rep in 1 2; do
  for v in rst new; do
    if [ $v = new ]; then unset FDG_DBG_LIB; else export FDG_DBG_LIB=variants/libfdg_$v.so; fi
    echo "== $v rep $rep" >> gpurun_out/s4p_ab.txt
    K=200 timeout 900 python scripts/ab.py "S=8,bm=11105995" "S=8,bm=11105995,cs=1" 2>&1 | grep us/batch >> gpurun_out/s4p_ab.txt
  done
done
