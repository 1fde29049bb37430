CFG=products K=300 timeout 900 python scripts/ab.py "S=8" "S=8,pipeline_gather_impl=4" "S=8,gather_pf64=0" "S=8,gather_pf64=1" "S=8,pipeline_gather_impl=4,gather_pf64=1" "S=8,pipeline_gather_impl=0" > gpurun_out/r2g_ab_products.txt 2>&1
CFG=papers K=300 timeout 900 python scripts/ab.py "S=8" "S=8,mode=sample" "S=8,mode=extract" "S=10" "S=6" > gpurun_out/r2g_ab_papers.txt 2>&1
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/r2g_bench20.json 2> gpurun_out/r2g_bench20.err
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_mt -c 40 --csv --log-file gpurun_out/r2g_mt.csv python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-per-call > /dev/null 2>&1
