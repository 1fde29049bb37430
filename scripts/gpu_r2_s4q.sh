# How far the samplers run ahead (per-batch output slots): config 3 and Papers.
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "pipeline_runner" > gpurun_out/s4q_tests.txt 2>&1; echo "rc=$?" >> gpurun_out/s4q_tests.txt
for rep in 1 2; do
  K=200 timeout 900 python scripts/ab.py "S=8,bm=11105995" "S=8,bm=11105995,pipe_slots=4" "S=8,bm=11105995,pipe_slots=8" "S=8,bm=11105995,pipe_slots=12" 2>&1 | grep us/batch >> gpurun_out/s4q_ab.txt
done
K=300 timeout 900 python scripts/ab.py "S=8" "S=8,pipe_slots=8" "S=8,pipe_slots=12" "S=8,pipe_slots=24" 2>&1 | grep us/batch >> gpurun_out/s4q_ab.txt
