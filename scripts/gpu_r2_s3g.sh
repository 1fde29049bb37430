# Buffer manager: reference counts inside the 16-byte slot records (one random record per
# hit / bind / release), and 64-byte L2 fills on the random metadata reads.
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/ -q -x -m gpu > gpurun_out/s3g_tests.txt 2>&1; echo "rc=$?" >> gpurun_out/s3g_tests.txt
for rep in 1 2; do
  for v in bmbase bmnohint new; do
    if [ $v = new ]; then unset FDG_DBG_LIB; else export FDG_DBG_LIB=variants/libfdg_$v.so; fi
    echo "== papers_bm $v rep $rep" >> gpurun_out/s3g_ab.txt
    K=200 timeout 900 python scripts/ab.py "S=8,bm=11105995" 2>&1 | grep us/batch >> gpurun_out/s3g_ab.txt
  done
done
unset FDG_DBG_LIB
FDG_PROFILE_RANGE=1 K=60 timeout 900 ncu --replay-mode app-range \
    --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct --csv \
    --log-file gpurun_out/s3g_range_bm.csv python scripts/ab.py "S=8,bm=11105995" > /dev/null 2>&1
