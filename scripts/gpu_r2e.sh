FDG_DBG_LIB=scripts/dbg/libfdg.so python scripts/dbg/rej_debug.py > gpurun_out/r2e_rej.txt 2>&1
timeout 1200 python -m pytest tests/test_cpp_shim.py tests/test_gpu_dataset.py tests/test_gpu_scale.py -q -m gpu 2>&1 | tail -30 > gpurun_out/r2e_tests.txt
./tools/set_loop --generate 111059956:128:16:7 4444000 50 > gpurun_out/r2e_perloop.txt 2>&1
