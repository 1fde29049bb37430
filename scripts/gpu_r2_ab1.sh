mkdir -p gpurun_out
K=300 timeout 900 python scripts/ab.py "S=8" "S=8,sampler_ctas_per_sm=2" "S=8,sampler_ctas_per_sm=4" "S=8,sampler_ctas_per_sm=8" \
  "S=8,mode=sample,sampler_ctas_per_sm=4" "S=8,mode=sample,sampler_ctas_per_sm=8" "S=8,mode=sample,mt_adaptive=0" "S=8,mt_adaptive=0" \
  "S=12" "S=12,mode=sample" "S=16,mode=sample" > gpurun_out/ab1.txt 2>&1
