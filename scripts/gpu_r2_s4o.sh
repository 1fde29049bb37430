# Config 3: extraction streams (metadata + move) above the samplers' priority, repeated.
mkdir -p gpurun_out
for rep in 1 2 3; do
  K=200 timeout 900 python scripts/ab.py "S=8,bm=11105995" "S=8,bm=11105995,extract_prio=1" "S=8,bm=11105995,cs=1" "S=8,bm=11105995,cs=1,extract_prio=1" 2>&1 | grep us/batch >> gpurun_out/s4o_ab.txt
done
