# Sampler kernels' CTA cap per SM (grid = min(work, SMs x cap / batches in the group)).
mkdir -p gpurun_out
for rep in 1 2; do
  K=300 timeout 900 python scripts/ab.py "S=8" "S=8,sampler_ctas_per_sm=8" "S=8,sampler_ctas_per_sm=12" "S=8,sampler_ctas_per_sm=24" "S=8,cs=1" "S=8,cs=1,sampler_ctas_per_sm=12" "S=8,cs=1,sampler_ctas_per_sm=24" 2>&1 | grep us/batch >> gpurun_out/s5a_ab.txt
done
