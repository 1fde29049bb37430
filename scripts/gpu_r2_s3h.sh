# Sampler: 64-byte L2 fills on the random CSR reads (sampnohint = plain loads), and the
# products gather's DRAM reads per engine (TMA bulk copies included).
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x > gpurun_out/s3h_tests.txt 2>&1; echo "rc=$?" >> gpurun_out/s3h_tests.txt
for cfg in papers products; do
  for rep in 1 2; do
    for v in sampnohint new; do
      if [ $v = new ]; then unset FDG_DBG_LIB; else export FDG_DBG_LIB=variants/libfdg_$v.so; fi
      echo "== $cfg $v rep $rep" >> gpurun_out/s3h_ab.txt
      CFG=$cfg K=300 timeout 600 python scripts/ab.py "S=8" "S=8,mode=sample" "S=8,cs=1" 2>&1 | grep us/batch >> gpurun_out/s3h_ab.txt
    done
  done
done
unset FDG_DBG_LIB
FDG_PROFILE_RANGE=1 K=100 timeout 600 ncu --replay-mode app-range \
    --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct --csv \
    --log-file gpurun_out/s3h_range_sample.csv python scripts/ab.py "S=8,mode=sample" > /dev/null 2>&1
SHORT=1 timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --csv \
  -k regex:gather --log-file gpurun_out/s3h_products_traffic.csv python scripts/products_traffic.py > gpurun_out/s3h_products_traffic.log 2>&1
