# C++ drop-in: sample_khop without the per-call zero fill of the bound (parity + per-call loop).
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_cpp_shim.py tests/test_session.py -q -x > gpurun_out/s5d_tests.txt 2>&1; echo "rc=$?" >> gpurun_out/s5d_tests.txt
for i in 1 2 3; do
  timeout 600 tools/set_loop --generate 111059956:128:16:7 4444000 200 2>&1 | grep per_call >> gpurun_out/s5d_percall.txt
done
