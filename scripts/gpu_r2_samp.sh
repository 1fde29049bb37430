# Sampler diagnosis: sample-only / extract-only / full timings vs sampler count, and DRAM bytes
# per batch of sample-only runs (ncu application-range replay) at S = 1, 2, 4, 8.
mkdir -p gpurun_out
K=300 timeout 900 python scripts/ab.py "S=8" "S=8,mode=sample" "S=8,mode=extract" "S=1,mode=sample" "S=2,mode=sample" \
   "S=4,mode=sample" "S=4" "S=2" > gpurun_out/samp_ab.txt 2>&1
for S in 1 2 4 8; do
  FDG_PROFILE_RANGE=1 K=100 timeout 600 ncu --replay-mode app-range \
    --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct --csv \
    --log-file gpurun_out/samp_range_S$S.csv python scripts/ab.py "S=$S,mode=sample" > /dev/null 2>&1
done
K=60 timeout 900 ncu --cache-control none --clock-control none -s 200 -c 120 \
  --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct \
  --csv --log-file gpurun_out/samp_kernels_S1.csv python scripts/ab.py S=1,mode=sample > /dev/null 2>&1
