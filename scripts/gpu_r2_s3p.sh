# Config 3: non-persistent row move (CTAs retire during the move) and the metadata stream at
# the samplers' priority.
mkdir -p gpurun_out
for rep in 1 2; do
  K=200 timeout 900 python scripts/ab.py "S=8,bm=11105995" "S=8,bm=11105995,bm_move_grid=1" "S=8,bm=11105995,bm_meta_prio=1" "S=8,bm=11105995,bm_move_grid=1,bm_meta_prio=1" 2>&1 | grep us/batch >> gpurun_out/s3p_ab.txt
done
