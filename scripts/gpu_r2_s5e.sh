# Seeds + layer 0 fused (k_early) re-measured with the final sampler (Bloom filter, lean passes).
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "early" > gpurun_out/s5e_tests.txt 2>&1; echo "rc=$?" >> gpurun_out/s5e_tests.txt
for rep in 1 2 3; do
  K=300 timeout 900 python scripts/ab.py "S=8" "S=8,early_fused=1" "S=8,cs=1" "S=8,cs=1,early_fused=1" 2>&1 | grep us/batch >> gpurun_out/s5e_ab.txt
done
CFG=products K=196 timeout 900 python scripts/ab.py "S=8" "S=8,early_fused=1" 2>&1 | grep us/batch >> gpurun_out/s5e_ab.txt
