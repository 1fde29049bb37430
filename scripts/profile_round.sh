# Round profiles: launch list of the bench command, ncu --set full of the two extraction
# kernels (device-resident gather, fused gather + trainer checksum), DRAM traffic per config.
set -x
ncu --metrics gpu__time_duration.sum --clock-control none -s 400 -c 400 --csv --log-file gpurun_out/launches.csv \
    python bench.py --steps 60 --warmup 5 --no-cpu-baseline > gpurun_out/launches_bench.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:k_gather16_dyn -s 10 -c 2 -o gpurun_out/gather16_full \
    python bench.py --steps 20 --warmup 5 --no-cpu-baseline > /dev/null 2>&1
ncu --set full --import-source on --clock-control none -k regex:k_gather_hash_rb -s 10 -c 2 -o gpurun_out/gather_hash_full \
    python bench.py --steps 20 --warmup 5 --no-cpu-baseline > /dev/null 2>&1
for c in papers friendster products; do
  ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
      -k regex:"k_gather16_dyn|k_gather_hash_rb" -s 6 -c 8 --csv --log-file gpurun_out/traffic_$c.csv \
      python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
done
