timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
S="python bench.py --dims 128,128,128 --profile-steps 1"
$S > gpurun_out/plain_small.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"stencil5_kernel" -c 1 -o gpurun_out/prof_st4 -f $S > gpurun_out/ncu_st4.log 2>&1
timeout 900 python bench.py --steps 4 --warmup 3 --no-cpu > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err
echo done
