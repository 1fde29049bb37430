# ncu --set full of the e2e path's fused gather + checksum inside the pipelined Papers run.
mkdir -p gpurun_out
K=40 timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_gather_hash_rb" -s 20 -c 1 \
  -o gpurun_out/s4z_hash_rb_full python scripts/ab.py "S=8,cs=1" > /dev/null 2>&1
