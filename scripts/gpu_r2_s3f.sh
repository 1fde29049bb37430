# DRAM bytes per random access (granularity limit x prefetch hints), and the products gather's
# read amplification under the same settings.
mkdir -p gpurun_out
timeout 300 scripts/probes/rand_gran > gpurun_out/s3f_rand_gran.txt 2>&1
timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sectors_srcunit_tex.sum,lts__t_requests_srcunit_tex.sum --csv \
  -k regex:k_rand --log-file gpurun_out/s3f_rand_gran_ncu.csv scripts/probes/rand_gran > /dev/null 2>&1
timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --csv \
  -k regex:gather --log-file gpurun_out/s3f_products_traffic.csv python scripts/products_traffic.py > gpurun_out/s3f_products_traffic.log 2>&1
