# Config 3's e2e path: row move + trainer checksum in one pass (k_move_hash_rb) vs move then
# a second pass over the slots.
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_scale.py -q -x -k "buffer_manager or extractor or bm or pipeline or scale" > gpurun_out/s3x_tests.txt 2>&1; echo "rc=$?" >> gpurun_out/s3x_tests.txt
for rep in 1 2; do
  K=200 timeout 900 python scripts/ab.py "S=8,bm=11105995,cs=1" "S=8,bm=11105995,cs=1,bm_move_hash=0" 2>&1 | grep us/batch >> gpurun_out/s3x_ab.txt
done
