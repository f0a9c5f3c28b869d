# c4 full size: per-launch DRAM traffic + time of the step's heavy kernels (single-pass metrics, no replay)
S="python bench.py --profile-steps 1"
$S > gpurun_out/plain_c4.log 2>&1 && \
ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active,lts__t_sector_hit_rate.pct \
    --clock-control none -k regex:"gemm_nn|gemm_tn|stencil5|reconstruct_dmma" -c 12 --csv \
    --log-file gpurun_out/c4_metrics.csv $S > gpurun_out/ncu_c4.log 2>&1
C="python bench.py --profile-steps 2"
$C > gpurun_out/plain_c4b.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c4.csv $C > gpurun_out/ncu_launch.log 2>&1
echo done
