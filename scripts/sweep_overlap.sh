# dynamic row-group gather (gather_impl=4) inside the pipelines
for c in papers friendster; do
CFG=$c timeout 600 python scripts/ab.py "S=8" "S=8,gather_impl=4,rb_ctas_per_sm=1" "S=8,gather_impl=4,rb_ctas_per_sm=2" "S=8,gather_impl=4,rb_ctas_per_sm=1,extract_streams=1" "S=8,gather_impl=4,rb_ctas_per_sm=2,extract_streams=1" "S=8,mode=extract,gather_impl=4,rb_ctas_per_sm=2"
done
