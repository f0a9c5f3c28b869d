mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_emit.py tests/test_gpu_update_and_solve.py tests/test_gpu_ozaki.py -q -x > gpurun_out/emit_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/emit_tests.log
timeout 900 python bench.py --no-cpu > gpurun_out/emit_bench_c4.json 2> gpurun_out/emit_bench_c4.err
SWB_EMIT=0 timeout 900 python bench.py --no-cpu --no-e2e > gpurun_out/noemit_bench_c4.json 2>> gpurun_out/emit_bench_c4.err
tail -25 gpurun_out/emit_tests.log; tail -3 gpurun_out/emit_bench_c4.err
for f in emit_bench_c4 noemit_bench_c4; do
python -c "import json;d=json.load(open('gpurun_out/$f.json'));p=d['phases_ms'];print('$f',round(d['ms_per_step'],1),d['clocks']['sm_mhz'],round(p['project'],2),round(p['rotate_split'],2),round(p['rotate_gemm'],2),round(p['rotate_join'],2),round(p['stencil'],2))"; done
