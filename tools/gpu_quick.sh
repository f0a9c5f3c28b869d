mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_ozaki.py tests/test_gpu_update_and_solve.py -q -x > gpurun_out/q_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/q_tests.log
timeout 900 python bench.py --no-cpu > gpurun_out/q_bench_c4.json 2> gpurun_out/q_bench_c4.err
tail -2 gpurun_out/q_tests.log
python -c "import json;d=json.load(open('gpurun_out/q_bench_c4.json'));p=d['phases_ms'];print(d['ms_per_step'],d['clocks']['sm_mhz'],round(p['rotate_split'],2),round(p['rotate_gemm'],2),round(p['rotate_join'],2),round(p['project'],2),round(p['stencil'],2))"
