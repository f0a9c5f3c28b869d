# per-launch durations of one c4 step (plus setup) -- ncu launch list
C="python bench.py --profile-steps 1 ${EXTRA:-}"
$C > gpurun_out/plain_launch.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launch_list.csv $C > gpurun_out/ncu_launch.log 2>&1
echo rc=$?
