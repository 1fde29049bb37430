for v in "" mb2 mb3 mb4; do
  lib=""; [ -n "$v" ] && lib=scripts/dbg/libfdg_$v.so
  echo "== variant ${v:-base}" >> gpurun_out/r2i_ab.txt
  FDG_DBG_LIB=$lib CFG=papers K=300 timeout 900 python scripts/ab.py "S=8" "S=8,mode=sample,mt_adaptive=0" >> gpurun_out/r2i_ab.txt 2>&1
done
