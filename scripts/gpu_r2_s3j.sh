# Config 3: k_move's register footprint (60 regs x 2 x 512 threads = 94% of the register file
# kept the samplers, the MT prefetch and the metadata chain off the SMs during every move).
mkdir -p gpurun_out
for rep in 1 2; do
  for v in new mv32 mv40 mv1 mv32r2 mv32c3; do
    if [ $v = new ]; then unset FDG_DBG_LIB; else export FDG_DBG_LIB=variants/libfdg_$v.so; fi
    echo "== papers_bm $v rep $rep" >> gpurun_out/s3j_ab.txt
    K=200 timeout 900 python scripts/ab.py "S=8,bm=11105995" 2>&1 | grep us/batch >> gpurun_out/s3j_ab.txt
  done
done
