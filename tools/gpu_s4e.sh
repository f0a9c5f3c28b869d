mkdir -p gpurun_out
export PYTHONPATH=$PWD
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/s4e_gpu_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/s4e_gpu_tests.log
tail -3 gpurun_out/s4e_gpu_tests.log
for c in c1 c2; do timeout 300 python bench.py --config $c --graph --no-cpu --no-e2e 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read());print('$c graph',d['ms_per_step'])"; done
for c in c3 c5; do timeout 300 python bench.py --config $c --no-cpu --no-e2e 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read());print('$c',d['ms_per_step'])"; done
timeout 900 python bench.py --no-cpu > gpurun_out/s4e_bench_c4.json 2> gpurun_out/s4e_bench_c4.err
python -c "import json;d=json.load(open('gpurun_out/s4e_bench_c4.json'));print(d['ms_per_step'],d['clocks']['sm_mhz'],{k:round(v,2) for k,v in d['phases_ms'].items() if v>0.5})"
