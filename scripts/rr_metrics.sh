M=dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sectors_op_atom.sum,lts__t_sectors_op_read.sum,lts__t_sectors_op_write.sum,lts__t_sector_op_atom_hit_rate.pct,lts__t_sector_op_read_hit_rate.pct,lts__t_sector_op_write_hit_rate.pct,gpu__time_duration.sum,lts__t_sectors_srcunit_tex_lookup_miss.sum
for m in "full 1 3" "sample 1 3" "extract 1 3"; do
FDG_PROFILE_RANGE=1 timeout 600 ncu --replay-mode app-range --clock-control none --metrics $M --csv python scripts/range_run.py $m > gpurun_out/rr_${m// /_}.csv 2>gpurun_out/rr_${m// /_}.err
done
