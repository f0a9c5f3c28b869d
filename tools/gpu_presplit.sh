mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_update_and_solve.py tests/test_gpu_capture.py tests/test_gpu_pipeline.py -q -x > gpurun_out/ps_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/ps_tests.log
tail -2 gpurun_out/ps_tests.log
for v in 1 0 1 0; do
SWB_PRESPLIT=$v timeout 600 python bench.py --no-cpu --no-e2e > gpurun_out/ps_$v.json 2>/dev/null
python -c "import json;d=json.load(open('gpurun_out/ps_$v.json'));p=d['phases_ms'];print('presplit=$v',round(d['ms_per_step'],1),d['clocks']['sm_mhz'],round(p['solve_prefill'],2),round(p['solve_system'],2),round(p['rotate_split'],2),round(p['rotate_gemm']+p['rotate_join'],2))"
done
