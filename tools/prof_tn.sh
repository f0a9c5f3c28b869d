timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
timeout 900 python bench.py --steps 4 --warmup 3 --no-cpu > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err
S="python bench.py --dims 256,256,128 --profile-steps 1"
$S > gpurun_out/plain_tn.log 2>&1 && \
ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active \
    --clock-control none -k regex:"gemm_tn" -s 2 -c 1 --csv --log-file gpurun_out/tn_metrics.csv $S > gpurun_out/ncu_tn.log 2>&1
echo done
