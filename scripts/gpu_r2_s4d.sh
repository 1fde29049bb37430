# Stream priorities: samplers high (default), all equal (flags 8), extraction high.
mkdir -p gpurun_out
for rep in 1 2; do
  K=300 timeout 900 python scripts/ab.py "S=8" "S=8,flags=8" "S=8,extract_prio=1" "S=8,cs=1" "S=8,cs=1,extract_prio=1" 2>&1 | grep us/batch >> gpurun_out/s4d_ab.txt
done
CFG=products K=196 timeout 900 python scripts/ab.py "S=8" "S=8,extract_prio=1" 2>&1 | grep us/batch >> gpurun_out/s4d_ab.txt
K=200 timeout 900 python scripts/ab.py "S=8,bm=11105995" "S=8,bm=11105995,extract_prio=1" 2>&1 | grep us/batch >> gpurun_out/s4d_ab.txt
