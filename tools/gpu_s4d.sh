mkdir -p gpurun_out
export PYTHONPATH=$PWD
timeout 600 compute-sanitizer --tool racecheck python -m pytest tests/test_gpu_parity.py -x -q -k "column_owner" > gpurun_out/s4d_race.log 2>&1; echo "race rc=$?" >> gpurun_out/s4d_race.log
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_capture.py tests/test_gpu_pipeline.py -x -q > gpurun_out/s4d_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/s4d_tests.log
timeout 300 python tools/small_lu_bench.py > gpurun_out/s4d_small_lu.log 2>&1
timeout 600 python bench.py --config c1 --graph --no-cpu > gpurun_out/s4d_bench_c1_graph.json 2> gpurun_out/s4d_bench_c1.err
tail -4 gpurun_out/s4d_race.log; tail -3 gpurun_out/s4d_tests.log; tail -12 gpurun_out/s4d_small_lu.log
python -c "import json;d=json.load(open('gpurun_out/s4d_bench_c1_graph.json'));print(d['ms_per_step'],d['clocks'])"
