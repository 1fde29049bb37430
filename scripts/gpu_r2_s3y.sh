# Config 3 plain move: row-group engine (k_move_hash_rb without the hash) vs k_move.
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "buffer_manager" > gpurun_out/s3y_tests.txt 2>&1; echo "rc=$?" >> gpurun_out/s3y_tests.txt
for rep in 1 2; do
  K=200 timeout 900 python scripts/ab.py "S=8,bm=11105995" "S=8,bm=11105995,bm_move_impl=2" "S=8,bm=11105995,bm_move_impl=2,hash_ctas_per_sm=2" 2>&1 | grep us/batch >> gpurun_out/s3y_ab.txt
done
