ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sectors_srcunit_tex_op_read.sum --clock-control none -k regex:k_gather -c 20 --csv --log-file gpurun_out/r2r_products_traffic.csv python scripts/products_traffic.py > gpurun_out/r2r.log 2>&1
HOST=1 BM=11105995 K=12 python scripts/trace_pipeline.py 8 > gpurun_out/r2r_host_trace.txt 2>&1
