set -x
S="python bench.py --dims 128,128,128 --profile-steps 1"
$S > gpurun_out/plain_small.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"stencil_kernel|reconstruct_kernel" -c 2 -o gpurun_out/prof_mem -f $S > gpurun_out/ncu_mem.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"gemm_" -s 4 -c 2 -o gpurun_out/prof_gemm -f $S > gpurun_out/ncu_gemm.log 2>&1
C="python bench.py --profile-steps 2"
$C > gpurun_out/plain_c4.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c4.csv $C > gpurun_out/ncu_launch.log 2>&1
echo done
