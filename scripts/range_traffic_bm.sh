# Whole-step DRAM traffic of the config-3 pipelined run (ncu application-range replay over
# K batches per range; ab.py runs three ranges): bytes per batch for step_roofline.
FDG_PROFILE_RANGE=1 K=50 timeout 1500 ncu --replay-mode app-range \
  --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --csv \
  --log-file gpurun_out/range_papers_bm.csv python scripts/ab.py S=8,bm=11105995 > gpurun_out/range_papers_bm.log 2>&1
