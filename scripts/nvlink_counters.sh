#!/bin/bash
# NVLink evidence for the row-sharded gather (needs >= 2 GPUs; one process, so ncu may wrap it):
# per-launch time and NVLink receive / transmit bytes of the gather kernel reading remote shards.
G=${1:-2}
ncu --query-metrics 2>/dev/null | grep -i -E "^nvl" > gpurun_out/nvlink_metric_names.txt
python scripts/nvlink_gather.py $G > gpurun_out/nvlink_gather_G$G.txt 2>&1
ncu --metrics gpu__time_duration.sum,nvlrx__bytes.sum,nvltx__bytes.sum,dram__bytes_read.sum --clock-control none \
    -k regex:k_gather -c 6 --csv --log-file gpurun_out/nvlink_counters_G$G.csv python scripts/nvlink_gather.py $G \
    > /dev/null 2>&1
