# Round-2 measurement pass 2: C4 proxy, out-of-core tier, train stage, whole-step DRAM traffic
# (range replay) for configs 2 and 3, full captures of the dominant kernels.
mkdir -p gpurun_out
timeout 1200 python bench.py --config mag --steps 200 --warmup 10 --no-per-call > gpurun_out/s3u_bench_mag.json 2> gpurun_out/s3u_bench_mag.err
timeout 1200 python bench.py --config papers_host_bm --steps 20 --warmup 5 > gpurun_out/s3u_bench_papers_host_bm.json 2> gpurun_out/s3u_bench_papers_host_bm.err
timeout 1200 python bench.py --train --steps 200 --warmup 10 --no-per-call --no-cpu-baseline > gpurun_out/s3u_bench_papers_train.json 2> gpurun_out/s3u_bench_papers_train.err
FDG_PROFILE_RANGE=1 K=50 timeout 900 ncu --replay-mode app-range \
  --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --csv \
  --log-file gpurun_out/s3u_range_papers.csv python scripts/ab.py S=8 > /dev/null 2>&1
FDG_PROFILE_RANGE=1 K=50 timeout 900 ncu --replay-mode app-range \
  --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --csv \
  --log-file gpurun_out/s3u_range_papers_bm.csv python scripts/ab.py S=8,bm=11105995 > /dev/null 2>&1
K=40 timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_gather16_dyn" -s 20 -c 1 \
  -o gpurun_out/s3u_gather16_dyn_full python scripts/ab.py S=8 > /dev/null 2>&1
K=40 timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_move|k_acquire|k_bind" -s 30 -c 3 \
  -o gpurun_out/s3u_bm_full python scripts/ab.py S=8,bm=11105995 > /dev/null 2>&1
