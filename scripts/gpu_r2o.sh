timeout 900 python bench.py --config papers_host_bm --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/r2o_hostbm.json 2> gpurun_out/r2o_hostbm.err
CFG=papers_host_bm K=40 timeout 900 python scripts/ab.py "S=8,bm=11105995" "S=8,bm=11105995,bm_overlap=0" > gpurun_out/r2o_ab.txt 2>&1
