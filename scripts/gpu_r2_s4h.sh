# Re-sweep of sampler count / grouping after the sampler changes (Papers, products, e2e form).
mkdir -p gpurun_out
K=300 timeout 900 python scripts/ab.py "S=8" "S=6" "S=10" "S=12" "S=8,G=2" "S=8,cs=1" "S=10,cs=1" "S=6,cs=1" 2>&1 | grep us/batch >> gpurun_out/s4h_ab.txt
CFG=products K=196 timeout 900 python scripts/ab.py "S=8" "S=6" "S=10" 2>&1 | grep us/batch >> gpurun_out/s4h_ab.txt
K=200 timeout 900 python scripts/ab.py "S=8,bm=11105995" "S=6,bm=11105995" "S=4,bm=11105995" 2>&1 | grep us/batch >> gpurun_out/s4h_ab.txt
