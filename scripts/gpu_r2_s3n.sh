# Hardware work queues: the runner drives 19 streams (8 samplers, 8 MT prefetch, 2 extraction,
# train) over CUDA_DEVICE_MAX_CONNECTIONS (default 8) queues -- false dependencies between them?
mkdir -p gpurun_out
for c in 8 16 32; do
  echo "== connections $c" >> gpurun_out/s3n_ab.txt
  CUDA_DEVICE_MAX_CONNECTIONS=$c K=300 timeout 600 python scripts/ab.py "S=8" "S=8,cs=1" "S=8,mode=sample" 2>&1 | grep us/batch >> gpurun_out/s3n_ab.txt
  CUDA_DEVICE_MAX_CONNECTIONS=$c K=200 timeout 600 python scripts/ab.py "S=8,bm=11105995" 2>&1 | grep us/batch >> gpurun_out/s3n_ab.txt
  CUDA_DEVICE_MAX_CONNECTIONS=$c CFG=products K=196 timeout 600 python scripts/ab.py "S=8" "S=8,cs=1" 2>&1 | grep us/batch >> gpurun_out/s3n_ab.txt
done
