mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_update_and_solve.py tests/test_gpu_bench_configs.py tests/test_gpu_capture.py tests/test_gpu_pipeline.py tests/test_oracle_golden.py -q -x > gpurun_out/sm_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/sm_tests.log
tail -3 gpurun_out/sm_tests.log
for c in c1 c2; do
timeout 600 python bench.py --config $c --graph --no-cpu --no-e2e > gpurun_out/sm_$c.json 2>/dev/null
python -c "import json;d=json.load(open('gpurun_out/sm_$c.json'));print('$c',d['ms_per_step'])"
done
