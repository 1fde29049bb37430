# Buffer manager: fused select + bind (parity + A/B); host tier with THP + NUMA-local pages.
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "buffer_manager or extractor or u64 or bm" > gpurun_out/s3v_tests.txt 2>&1; echo "rc=$?" >> gpurun_out/s3v_tests.txt
for rep in 1 2; do
  K=200 timeout 900 python scripts/ab.py "S=8,bm=11105995" "S=8,bm=11105995,bm_fuse_bind=1" 2>&1 | grep us/batch >> gpurun_out/s3v_ab.txt
done
K=200 timeout 900 python scripts/ab.py "S=8,bm=11105995,mode=extract" "S=8,bm=11105995,mode=extract,bm_fuse_bind=1" 2>&1 | grep us/batch >> gpurun_out/s3v_ab.txt
timeout 1200 python bench.py --config papers_host_bm --steps 20 --warmup 5 --no-cpu-baseline --option host_tier_thp=1 > gpurun_out/s3v_bench_host_thp.json 2> gpurun_out/s3v_bench_host_thp.err
numactl -H > gpurun_out/s3v_numa.txt 2>&1; free -g >> gpurun_out/s3v_numa.txt
