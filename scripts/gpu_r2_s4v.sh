# the reference's run_sync_reference at the products shape, and the
# reference arm for products and config 3.
mkdir -p gpurun_out
timeout 1500 python bench.py --impl reference --config products --steps 64 --warmup 3 --sync-reference > gpurun_out/s4v_ref_products.json 2> gpurun_out/s4v_ref_products.err
timeout 1500 python bench.py --impl reference --config papers_bm --steps 16 --warmup 3 > gpurun_out/s4v_ref_papers_bm.json 2> gpurun_out/s4v_ref_papers_bm.err
