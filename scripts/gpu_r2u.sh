(nvidia-smi topo -m; lscpu | grep -i numa; for d in /sys/bus/pci/devices/*; do [ -f $d/class ] && grep -q 0x0302 $d/class && echo "$d numa=$(cat $d/numa_node)"; done; free -g) > gpurun_out/r2u_topo.txt 2>&1
python scripts/host_tier_gather.py 111059956 1 > gpurun_out/r2u_host_papers_local.txt 2>&1
