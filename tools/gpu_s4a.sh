# Session-4 health check: full GPU test suite, smoke, c4 bench (no CPU leg).
mkdir -p gpurun_out
export PYTHONPATH=$PWD
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/s4_gpu_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/s4_gpu_tests.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/s4_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/s4_smoke.log
timeout 900 python bench.py --no-cpu > gpurun_out/s4_bench_c4.json 2> gpurun_out/s4_bench_c4.err
tail -3 gpurun_out/s4_gpu_tests.log; cat gpurun_out/s4_smoke.log
python -c "import json;d=json.load(open('gpurun_out/s4_bench_c4.json'));print(d['ms_per_step'],d['clocks'],d['phases_ms'])"
