# Hardware queues: the synchronous per-call loop vs the pipeline at 8 / 16 / 32.
mkdir -p gpurun_out
for rep in 1 2; do
for c in 8 16 32; do
  echo "== connections $c" >> gpurun_out/s3t_percall.txt
  CUDA_DEVICE_MAX_CONNECTIONS=$c timeout 600 tools/set_loop --generate 111059956:128:16:7 4444000 50 2>&1 | grep per_call >> gpurun_out/s3t_percall.txt
done
done
for c in 16 32; do
  echo "== connections $c" >> gpurun_out/s3t_ab.txt
  CUDA_DEVICE_MAX_CONNECTIONS=$c K=300 timeout 600 python scripts/ab.py "S=8" "S=8,cs=1" "S=8,mode=sample" 2>&1 | grep us/batch >> gpurun_out/s3t_ab.txt
  CUDA_DEVICE_MAX_CONNECTIONS=$c CFG=products K=196 timeout 600 python scripts/ab.py "S=8" "S=8,cs=1" 2>&1 | grep us/batch >> gpurun_out/s3t_ab.txt
done
