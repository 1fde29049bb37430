# SM-side cost of the sampler chain (sample-only pipelined run, Papers shape): per kernel the
# duration, issued instructions, active-warp occupancy and SM / DRAM throughput.
K=60 timeout 900 ncu --cache-control none --clock-control none -s 200 -c 120 \
  --metrics gpu__time_duration.sum,smsp__inst_executed.sum,sm__warps_active.avg.pct_of_peak_sustained_active,sm__throughput.avg.pct_of_peak_sustained_elapsed,gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed,launch__grid_size,launch__registers_per_thread,smsp__average_warp_latency_issue_stalled_long_scoreboard.ratio,smsp__cycles_active.avg \
  --csv --log-file gpurun_out/sampler_sm.csv python scripts/ab.py S=8,mode=sample > /dev/null 2>&1
