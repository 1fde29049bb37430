# Early-table Bloom filter for the last layer's lookups: parity + A/B.
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "sample or pipeline" > gpurun_out/s4c_tests.txt 2>&1; echo "rc=$?" >> gpurun_out/s4c_tests.txt
for rep in 1 2; do
  K=300 timeout 900 python scripts/ab.py "S=8" "S=8,early_bloom=0" "S=8,mode=sample" "S=8,mode=sample,early_bloom=0" "S=8,cs=1" "S=8,cs=1,early_bloom=0" 2>&1 | grep us/batch >> gpurun_out/s4c_ab.txt
done
CFG=products K=196 timeout 900 python scripts/ab.py "S=8" "S=8,early_bloom=0" "S=8,mode=sample" "S=8,mode=sample,early_bloom=0" 2>&1 | grep us/batch >> gpurun_out/s4c_ab.txt
