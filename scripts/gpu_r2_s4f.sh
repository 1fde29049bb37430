# Last intern pass occupancy vs spills: 64 / 48 / 40 (default) registers.
mkdir -p gpurun_out
for rep in 1 2; do
  for v in il4 il5 new; do
    if [ $v = new ]; then unset FDG_DBG_LIB; else export FDG_DBG_LIB=variants/libfdg_$v.so; fi
    echo "== $v rep $rep" >> gpurun_out/s4f_ab.txt
    K=300 timeout 900 python scripts/ab.py "S=8" "S=8,mode=sample" "S=8,cs=1" 2>&1 | grep us/batch >> gpurun_out/s4f_ab.txt
    CFG=products K=196 timeout 900 python scripts/ab.py "S=8" 2>&1 | grep us/batch >> gpurun_out/s4f_ab.txt
  done
done
