# ncu --set full of the Papers layer-2 expansion and the final intern pass (host-API sample_khop calls)
mkdir -p gpurun_out
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_expand|k_intern_s" -s 8 -c 8 \
  -o gpurun_out/samp_full python scripts/sample_prof.py > gpurun_out/samp_full.log 2>&1
