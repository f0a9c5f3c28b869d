# Round-2 evidence after the wide-MMA rotation (gpurun, one GPU): GPU tests,
# the default bench line, then ncu (each under its own timeout): the c4 launch
# list of one step, DRAM traffic of the heavy kernels (capped launch counts).
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/r2c_gpu_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/r2c_gpu_tests.log
python bench.py > gpurun_out/r2c_bench_c4.json 2> gpurun_out/r2c_bench_c4.err; echo "bench rc=$?"
S="python bench.py --profile-steps 1"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv $S > gpurun_out/r2c_launches_c4.csv 2> gpurun_out/r2c_ncu_launch.err
echo "launch list rc=$? lines=$(wc -l < gpurun_out/r2c_launches_c4.csv)"
timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,lts__t_sector_hit_rate.pct \
    --clock-control none -k regex:"gemm_tn_sym_kernel|stencil5_kernel|reconstruct_dmma_kernel|oz_gemm_kernel|oz_slice_rows_kernel" \
    -c 14 --csv $S > gpurun_out/r2c_c4_metrics.csv 2> gpurun_out/r2c_ncu_metrics.err
echo "metrics rc=$? lines=$(wc -l < gpurun_out/r2c_c4_metrics.csv)"
tail -2 gpurun_out/r2c_gpu_tests.log
