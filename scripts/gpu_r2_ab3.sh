mkdir -p gpurun_out
K=300 timeout 900 python scripts/ab.py "S=8" "S=10" "S=12" "S=16" > gpurun_out/ab3.txt 2>&1
for v in minb3 last3 minb1; do echo "variant $v" >> gpurun_out/ab3.txt
FDG_DBG_LIB=variants/libfdg_$v.so K=300 timeout 900 python scripts/ab.py "S=8" "S=12" "S=8,mode=sample" >> gpurun_out/ab3.txt 2>&1; done
