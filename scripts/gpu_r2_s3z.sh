# Plain Papers pipeline gather: row-group engine at one CTA per SM vs the chunk-striped default.
mkdir -p gpurun_out
for rep in 1 2; do
  K=300 timeout 900 python scripts/ab.py "S=8" "S=8,pipeline_gather_impl=4,rb_ctas_per_sm=1" "S=8,pipeline_gather_impl=4,rb_ctas_per_sm=2" 2>&1 | grep us/batch >> gpurun_out/s3z_ab.txt
done
CFG=products K=196 timeout 900 python scripts/ab.py "S=8" "S=8,pipeline_gather_impl=4,rb_ctas_per_sm=1" 2>&1 | grep us/batch >> gpurun_out/s3z_ab.txt
CFG=friendster K=200 timeout 900 python scripts/ab.py "S=8" "S=8,pipeline_gather_impl=4,rb_ctas_per_sm=1" 2>&1 | grep us/batch >> gpurun_out/s3z_ab.txt
