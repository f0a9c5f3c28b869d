# select_m: GPU tests, per-round select_m timing (cooperative QR vs SWB_HH_COOP=0), c3 bench
mkdir -p gpurun_out
export PYTHONPATH=$PWD
timeout 600 python -m pytest tests/test_gpu_select.py tests/test_gpu_bench_configs.py -q -x > gpurun_out/sel_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/sel_tests.log
timeout 600 python tools/select_bench.py 5 > gpurun_out/sel_plain.log 2>&1
SWB_HH_COOP=0 timeout 600 python tools/select_bench.py 5 > gpurun_out/sel_plain_old.log 2>&1
timeout 600 python bench.py --config c3 --no-cpu > gpurun_out/sel_c3.json 2> gpurun_out/sel_c3.err
tail -2 gpurun_out/sel_tests.log; cat gpurun_out/sel_plain.log gpurun_out/sel_plain_old.log
python -c "import json;d=json.load(open('gpurun_out/sel_c3.json'));print(d['ms_per_step'],d['clocks']['sm_mhz'])"
