# Per-kernel DRAM traffic of the sampler chain (sample-only pipelined run, Papers shape).
K=60 timeout 900 ncu --cache-control none --clock-control none -s 200 -c 120 \
  --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct \
  --csv --log-file gpurun_out/sampler_traffic.csv python scripts/ab.py S=8,mode=sample > /dev/null 2>&1
