# TMA row move for the buffer manager (parity + A/B), then the fused checksum at 1 CTA/SM.
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "buffer_manager or bm or extractor" > gpurun_out/s3l_tests.txt 2>&1; echo "rc=$?" >> gpurun_out/s3l_tests.txt
for rep in 1 2; do
  echo "== papers_bm rep $rep" >> gpurun_out/s3l_ab.txt
  K=200 timeout 900 python scripts/ab.py "S=8,bm=11105995" "S=8,bm=11105995,bm_move_impl=1" 2>&1 | grep us/batch >> gpurun_out/s3l_ab.txt
done
K=200 timeout 900 python scripts/ab.py "S=8,bm=11105995,mode=extract" "S=8,bm=11105995,mode=extract,bm_move_impl=1" 2>&1 | grep us/batch >> gpurun_out/s3l_ab.txt
bash scripts/gpu_r2_s3k.sh
