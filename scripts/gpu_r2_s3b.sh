# ncu --set full of the sampler's kernels inside a sample-only pipelined Papers run (8 samplers,
# warm caches: --cache-control none), one batch's chain after 40 batches.
mkdir -p gpurun_out
K=60 timeout 900 ncu --set full --import-source on --cache-control none --clock-control none \
  -k regex:"k_expand|k_intern_s|k_fill_ones|k_seeds" -s 400 -c 10 \
  -o gpurun_out/s3b_samp_full python scripts/ab.py "S=8,mode=sample" > gpurun_out/s3b_samp_full.log 2>&1
CFG=products K=60 timeout 900 ncu --set full --import-source on --cache-control none --clock-control none \
  -k regex:"k_expand|k_intern_s|k_fill_ones|k_seeds" -s 400 -c 10 \
  -o gpurun_out/s3b_samp_full_products python scripts/ab.py "S=8,mode=sample" > gpurun_out/s3b_samp_full_products.log 2>&1
timeout 300 python -c "
import paper_2406_13984_b200 as fd
print('tc_write_hi', fd.featdrive.get_option('tc_write_hi'))" > gpurun_out/s3b_tc.txt 2>&1
