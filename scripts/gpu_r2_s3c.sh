# Fused gather + checksum (the e2e path's extraction): static vs dynamic row-group claims.
mkdir -p gpurun_out
K=300 timeout 600 python scripts/ab.py "S=8,cs=1" "S=8,cs=1,hash_dyn=1" "S=8,cs=1,mode=extract" "S=8,cs=1,mode=extract,hash_dyn=1" "S=8" "S=8,cs=1" "S=8,cs=1,hash_dyn=1" > gpurun_out/s3c_ab_papers.txt 2>&1
CFG=products K=196 timeout 600 python scripts/ab.py "S=8,cs=1" "S=8,cs=1,hash_dyn=1" "S=8" > gpurun_out/s3c_ab_products.txt 2>&1
CFG=friendster K=200 timeout 900 python scripts/ab.py "S=8,cs=1" "S=8,cs=1,hash_dyn=1" > gpurun_out/s3c_ab_friendster.txt 2>&1
