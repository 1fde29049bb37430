# row-group dynamic gather with 128-byte chunks (fewer registers) inside the pipelines
for c in papers friendster; do
CFG=$c timeout 600 python scripts/ab.py "S=8" "S=8,pipeline_gather_impl=4,rb_chunk=128,rb_ctas_per_sm=1" "S=8,pipeline_gather_impl=4,rb_chunk=128,rb_ctas_per_sm=2" "S=8,pipeline_gather_impl=4,rb_chunk=128,rb_ctas_per_sm=3" "S=8,mode=extract,pipeline_gather_impl=4,rb_chunk=128,rb_ctas_per_sm=2"
done
