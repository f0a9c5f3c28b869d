# stencil pass at c4: DRAM bytes / duration / L2 hit rate (single-pass metrics)
S="python bench.py --profile-steps 1 ${EXTRA:-}"
$S > gpurun_out/plain_std.log 2>&1 && \
ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct,lts__t_sectors_srcunit_tex_op_read.sum,lts__t_sectors_op_read.sum,sm__throughput.avg.pct_of_peak_sustained_elapsed \
    --clock-control none -k regex:stencil[56] -c 1 --csv --log-file gpurun_out/st_dram.csv $S > gpurun_out/ncu_std.log 2>&1
echo rc=$?
