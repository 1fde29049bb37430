# Sampler kernels after the Bloom filter: ncu (warm, serialised) of one batch's chain inside a
# sample-only pipelined run, Papers and products.
mkdir -p gpurun_out
K=60 timeout 900 ncu --set full --import-source on --cache-control none --clock-control none \
  -k regex:"k_expand|k_intern_s|k_fill_ones|k_seeds|k_replay" -s 440 -c 11 \
  -o gpurun_out/s4e_samp_full python scripts/ab.py "S=8,mode=sample" > gpurun_out/s4e_samp_full.log 2>&1
