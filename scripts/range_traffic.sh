# Whole-run DRAM traffic of the pipelined run (ncu application-range replay): does sampling
# next to the gather add DRAM traffic (hash tables thrashed out of L2)?
for spec in "S=6" "S=6,mode=extract" "S=6,mode=sample"; do
  FDG_PROFILE_RANGE=1 K=100 timeout 600 ncu --replay-mode app-range \
    --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct --csv \
    --log-file gpurun_out/range_$(echo $spec | tr ',=' '__').csv python scripts/ab.py "$spec" > /dev/null 2>&1
done
