# Round-end evidence for profiles/ (run under gpurun, 1 GPU): plain bench
# lines first (each exits 0 without ncu), then the ncu launch list of the
# same c4 step and one --set full capture of the dominant kernel.
mkdir -p gpurun_out
python bench.py > gpurun_out/fin_c4.json 2> gpurun_out/fin_c4.err; echo "c4 rc=$?"
python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/fin_ref.json 2> gpurun_out/fin_ref.err; echo "ref rc=$?"
python bench.py --config c5 > gpurun_out/fin_c5.json 2> gpurun_out/fin_c5.err; echo "c5 rc=$?"
C="python bench.py --profile-steps 1"
$C > gpurun_out/fin_plain_launch.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,dram__bytes_read.sum,dram__bytes_write.sum \
    --clock-control none --csv --log-file gpurun_out/fin_launch_list.csv $C > gpurun_out/fin_ncu_launch.log 2>&1; echo "launch list rc=$?"
ncu --set full --clock-control none --import-source on -k regex:oz_gemm_kernel -s 3 -c 1 -o gpurun_out/fin_oz_gemm $C \
    > gpurun_out/fin_ncu_oz.log 2>&1; echo "oz full rc=$?"
ncu --set full --clock-control none --import-source on -k regex:gemm_tn_sym_kernel -s 2 -c 1 -o gpurun_out/fin_tn_sym $C \
    > gpurun_out/fin_ncu_tn.log 2>&1; echo "tn full rc=$?"
