# Round-end evidence for profiles/ (run under gpurun; one ncu tool per command):
#  1. the bench command itself, plain (exit 0 first), then its ncu launch list
#  2. per-kernel DRAM traffic / tensor-pipe share of one c4 step's heavy kernels
set -e
python bench.py > gpurun_out/r1_bench_plain.json 2> gpurun_out/r1_bench_plain.err
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r1_launches_c4.csv \
    python bench.py > gpurun_out/r1_ncu_launch.log 2>&1
S="python bench.py --profile-steps 1"
ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,lts__t_sector_hit_rate.pct \
    --clock-control none -k regex:"gemm_nn_kernel|gemm_tn_sym_kernel|stencil5_kernel|reconstruct_dmma_kernel" --csv \
    --log-file gpurun_out/r1_c4_metrics.csv $S > gpurun_out/r1_ncu_metrics.log 2>&1
echo done
