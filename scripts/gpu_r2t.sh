cat /sys/kernel/mm/transparent_hugepage/enabled > gpurun_out/r2t_thp.txt 2>&1
python scripts/host_tier_gather.py 8000000 0 > gpurun_out/r2t_host_8m.txt 2>&1
python scripts/host_tier_gather.py 111059956 0 > gpurun_out/r2t_host_papers.txt 2>&1
python scripts/host_tier_gather.py 111059956 1 > gpurun_out/r2t_host_papers_thp.txt 2>&1
