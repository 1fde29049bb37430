mkdir -p gpurun_out
K=300 timeout 900 python scripts/ab.py "S=8" "S=8,mode=sample" > gpurun_out/ab5.txt 2>&1
for v in exp8; do echo "variant $v" >> gpurun_out/ab5.txt
FDG_DBG_LIB=variants/libfdg_$v.so K=300 timeout 900 python scripts/ab.py "S=8" "S=8,mode=sample" >> gpurun_out/ab5.txt 2>&1; done
K=100 timeout 300 python scripts/trace_pipeline.py 8 > gpurun_out/trace3_S8_full.txt 2>&1
