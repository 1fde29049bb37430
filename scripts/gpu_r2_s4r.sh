# Config 3 split row move: parity + A/B.
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "split_move or buffer_manager or pipeline_runner" > gpurun_out/s4r_tests.txt 2>&1; echo "rc=$?" >> gpurun_out/s4r_tests.txt
for rep in 1 2; do
  K=200 timeout 900 python scripts/ab.py "S=8,bm=11105995" "S=8,bm=11105995,bm_split_move=1" "S=8,bm=11105995,bm_split_move=1,extract_prio=0" 2>&1 | grep us/batch >> gpurun_out/s4r_ab.txt
done
