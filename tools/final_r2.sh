# Round-2 final evidence (gpurun, one GPU): GPU tests, smoke, bench lines for
# every config (c4 default with the CPU baseline, the reference arm, c1 / c2
# as CUDA-graph replays, c3, c5), the c4 launch list and one --set full
# capture of the rotation GEMM; each ncu leg under its own timeout.
mkdir -p gpurun_out
export PYTHONPATH=$PWD
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/g_gpu_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/g_gpu_tests.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/g_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/g_smoke.log
timeout 1200 python bench.py > gpurun_out/g_bench_c4.json 2> gpurun_out/g_bench_c4.err
timeout 900 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/g_bench_ref.json 2> gpurun_out/g_bench_ref.err
timeout 900 python bench.py --config c1 --graph > gpurun_out/g_bench_c1_graph.json 2> gpurun_out/g_bench_c1.err
timeout 900 python bench.py --config c2 --graph > gpurun_out/g_bench_c2_graph.json 2> gpurun_out/g_bench_c2.err
timeout 900 python bench.py --config c3 > gpurun_out/g_bench_c3.json 2> gpurun_out/g_bench_c3.err
timeout 900 python bench.py --config c5 > gpurun_out/g_bench_c5.json 2> gpurun_out/g_bench_c5.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv python bench.py --profile-steps 1 \
  > gpurun_out/g_launches_c4.csv 2> gpurun_out/g_ncu_launch.err; echo "launch list rc=$?"
timeout 600 ncu --set full --import-source on --clock-control none -k regex:oz_gemm_kernel -c 1 -f -o gpurun_out/g_oz_gemm \
  python tools/oz_bench.py 1048576 400 1 > gpurun_out/g_ncu_oz.log 2>&1; echo "oz full rc=$?"
tail -2 gpurun_out/g_gpu_tests.log; cat gpurun_out/g_smoke.log
for f in g_bench_c4 g_bench_c1_graph g_bench_c2_graph g_bench_c3 g_bench_c5; do
python -c "import json;d=json.load(open('gpurun_out/$f.json'));print('$f',round(d['ms_per_step'],3),d['value'],d['clocks']['sm_mhz'],(d.get('cpu_baseline') or {}).get('value'))"; done
cat gpurun_out/g_bench_ref.json
