# Round-2 evidence after the wide-MMA rotation (run under gpurun, one GPU):
# plain bench first (exits 0), then ncu over ONE c4 step: launch list,
# per-kernel DRAM traffic of the heavy kernels, one --set full capture of
# the top kernels (oz_gemm_kernel, gemm_tn_sym_kernel).
mkdir -p gpurun_out
python bench.py > gpurun_out/r2b_bench_plain.json 2> gpurun_out/r2b_bench_plain.err; echo "bench rc=$?"
S="python bench.py --profile-steps 1"
ncu --metrics gpu__time_duration.sum --clock-control none --csv $S > gpurun_out/r2b_launches_c4.csv 2> gpurun_out/r2b_ncu_launch.err
echo "launch list rc=$?"
ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,lts__t_sector_hit_rate.pct \
    --clock-control none -k regex:"gemm_tn_sym_kernel|stencil5_kernel|reconstruct_dmma_kernel|oz_gemm_kernel|oz_slice_rows_kernel" \
    --csv $S > gpurun_out/r2b_c4_metrics.csv 2> gpurun_out/r2b_ncu_metrics.err
echo "metrics rc=$?"
ncu --set full --import-source on --clock-control none -k regex:oz_gemm_kernel -s 3 -c 1 -f -o gpurun_out/r2b_oz_gemm $S \
    > gpurun_out/r2b_ncu_oz.log 2>&1; echo "oz full rc=$?"
