# Per-call SET loop regression check (hardware queues), fused early-layer sampler (parity + A/B).
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_cpp_shim.py tests/test_session.py tests/test_gpu_scale.py -q -x > gpurun_out/s3s_tests.txt 2>&1; echo "rc=$?" >> gpurun_out/s3s_tests.txt
for c in 8 32; do
  echo "== connections $c" >> gpurun_out/s3s_percall.txt
  CUDA_DEVICE_MAX_CONNECTIONS=$c timeout 600 tools/set_loop --generate 111059956:128:16:7 4444000 50 >> gpurun_out/s3s_percall.txt 2>&1
done
for rep in 1 2; do
  K=300 timeout 900 python scripts/ab.py "S=8" "S=8,early_fused=0" "S=8,mode=sample" "S=8,mode=sample,early_fused=0" "S=8,cs=1" "S=8,cs=1,early_fused=0" 2>&1 | grep us/batch >> gpurun_out/s3s_ab.txt
done
CFG=products K=196 timeout 900 python scripts/ab.py "S=8" "S=8,early_fused=0" "S=8,mode=sample" "S=8,mode=sample,early_fused=0" 2>&1 | grep us/batch >> gpurun_out/s3s_ab.txt
K=200 timeout 900 python scripts/ab.py "S=8,bm=11105995" "S=8,bm=11105995,early_fused=0" 2>&1 | grep us/batch >> gpurun_out/s3s_ab.txt
