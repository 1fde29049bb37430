# Config 3: batch j's move right after its bind (next to release j-1) vs after the release.
mkdir -p gpurun_out
for rep in 1 2; do
  K=200 timeout 900 python scripts/ab.py "S=8,bm=11105995" "S=8,bm=11105995,bm_move_early=1" "S=8,bm=11105995,cs=1" "S=8,bm=11105995,cs=1,bm_move_early=1" 2>&1 | grep us/batch >> gpurun_out/s4a_ab.txt
done
