# update_and_solve: GPU tests + c4 bench fused vs separate (gpurun, one GPU)
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_update_and_solve.py tests/test_gpu_ozaki.py -q -x > gpurun_out/fused_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/fused_tests.log
timeout 900 python bench.py --no-cpu > gpurun_out/fused_bench_c4.json 2> gpurun_out/fused_bench_c4.err
SWB_FUSED=0 timeout 900 python bench.py --no-cpu --no-e2e > gpurun_out/sep_bench_c4.json 2>> gpurun_out/fused_bench_c4.err
tail -15 gpurun_out/fused_tests.log; tail -5 gpurun_out/fused_bench_c4.err
for f in fused_bench_c4 sep_bench_c4; do
python -c "import json;d=json.load(open('gpurun_out/$f.json'));print('$f',d['ms_per_step'],d['solve'],d.get('e2e',{}).get('value'),d['clocks']['sm_mhz'],{k:round(v,3) for k,v in d['phases_ms'].items()})"; done
