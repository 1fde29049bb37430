# Lean next-frontier intern passes chosen by the runner for pipelines without the checksum.
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "pipeline or sample" > gpurun_out/s4x_tests.txt 2>&1; echo "rc=$?" >> gpurun_out/s4x_tests.txt
for rep in 1 2 3; do
  K=300 timeout 900 python scripts/ab.py "S=8" "S=8,intern_lean=0" "S=8,cs=1" "S=8,cs=1,intern_lean=0" 2>&1 | grep us/batch >> gpurun_out/s4x_ab.txt
  CFG=products K=196 timeout 900 python scripts/ab.py "S=8" "S=8,intern_lean=0" 2>&1 | grep us/batch >> gpurun_out/s4x_ab.txt
done
K=200 timeout 900 python scripts/ab.py "S=8,bm=11105995" "S=8,bm=11105995,intern_lean=0" 2>&1 | grep us/batch >> gpurun_out/s4x_ab.txt
