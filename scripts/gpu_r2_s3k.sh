# The e2e path's fused gather + checksum at one CTA per SM (124 registers x 256 threads: two
# CTAs filled the register file and kept the samplers off the SMs).
mkdir -p gpurun_out
for cfg in papers products friendster; do
  for rep in 1 2; do
    echo "== $cfg rep $rep" >> gpurun_out/s3k_ab.txt
    CFG=$cfg K=300 timeout 900 python scripts/ab.py "S=8,cs=1" "S=8,cs=1,hash_ctas_per_sm=1" "S=8" "S=8,cs=1,mode=extract,hash_ctas_per_sm=1" 2>&1 | grep us/batch >> gpurun_out/s3k_ab.txt
  done
done
