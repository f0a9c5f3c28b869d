mkdir -p gpurun_out
export PYTHONPATH=$PWD
timeout 900 python -m pytest tests/test_gpu_update_and_solve.py tests/test_gpu_registration.py -x -q > gpurun_out/s4b_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/s4b_tests.log
timeout 900 python bench.py --config c5 --no-cpu > gpurun_out/s4b_bench_c5.json 2> gpurun_out/s4b_bench_c5.err
tail -3 gpurun_out/s4b_tests.log
python -c "import json;d=json.load(open('gpurun_out/s4b_bench_c5.json'));print(d['ms_per_step'],d['clocks'],d['phases_ms'])"
