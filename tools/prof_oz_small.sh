# ncu sanity + the rotation GEMM's full capture on one 1M-row chunk (gpurun, one GPU)
mkdir -p gpurun_out
export PYTHONPATH=$PWD
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv python bench.py --config c1 --profile-steps 1 \
  > gpurun_out/r2b_launches_c1.csv 2> gpurun_out/r2b_launches_c1.err; echo "c1 launch list rc=$?"
timeout 600 ncu --set full --import-source on --clock-control none -k regex:oz_gemm_kernel -c 1 -f -o gpurun_out/r2b_oz_gemm \
  python tools/oz_bench.py 1048576 400 1 > gpurun_out/r2b_ncu_oz.log 2>&1; echo "oz full rc=$?"
tail -5 gpurun_out/r2b_ncu_oz.log
