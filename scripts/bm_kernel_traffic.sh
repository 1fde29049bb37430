# Per-kernel DRAM traffic / L2 hit rate of the buffer-manager kernels inside the config-3
# pipeline (extract-only, serial move so each kernel runs alone): which metadata kernel
# pays for random DRAM sectors.
K=40 timeout 900 ncu --cache-control none --clock-control none -k regex:'k_acquire|k_select|k_bind|k_release|k_move|k_compact' -s 60 -c 60 \
  --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,lts__t_sectors.sum,lts__t_requests.sum \
  --csv --log-file gpurun_out/bm_kernel_traffic.csv python scripts/ab.py S=8,bm=11105995,mode=extract,bm_overlap=0 > /dev/null 2>&1
