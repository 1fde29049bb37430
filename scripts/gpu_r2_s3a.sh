# Session-3 state of the sampler: sample-only / extract-only / full timings (Papers, products)
# and DRAM bytes per batch of the sample-only and full runs (ncu application-range replay).
mkdir -p gpurun_out
K=300 timeout 600 python scripts/ab.py "S=8" "S=8,mode=sample" "S=8,mode=extract" > gpurun_out/s3a_ab_papers.txt 2>&1
CFG=products K=196 timeout 600 python scripts/ab.py "S=8" "S=8,mode=sample" "S=8,mode=extract" > gpurun_out/s3a_ab_products.txt 2>&1
for spec in "S=8,mode=sample" "S=8"; do
  FDG_PROFILE_RANGE=1 K=100 timeout 600 ncu --replay-mode app-range \
    --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct --csv \
    --log-file gpurun_out/s3a_range_papers_$(echo $spec | tr ',=' '__').csv python scripts/ab.py "$spec" > /dev/null 2>&1
  FDG_PROFILE_RANGE=1 CFG=products K=100 timeout 600 ncu --replay-mode app-range \
    --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct --csv \
    --log-file gpurun_out/s3a_range_products_$(echo $spec | tr ',=' '__').csv python scripts/ab.py "$spec" > /dev/null 2>&1
done
