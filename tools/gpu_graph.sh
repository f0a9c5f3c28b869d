mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_capture.py tests/test_gpu_update_and_solve.py -q -x > gpurun_out/graph_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/graph_tests.log
timeout 600 python bench.py --config c1 --no-cpu --graph > gpurun_out/graph_bench_c1.json 2> gpurun_out/graph_bench_c1.err
timeout 600 python bench.py --config c2 --no-cpu --graph > gpurun_out/graph_bench_c2.json 2>> gpurun_out/graph_bench_c1.err
tail -15 gpurun_out/graph_tests.log; tail -5 gpurun_out/graph_bench_c1.err
for f in graph_bench_c1 graph_bench_c2; do
python -c "import json;d=json.load(open('gpurun_out/$f.json'));print('$f',d['ms_per_step'],d['e2e']['ms_per_step'],d['gpu_launches'],d['steps'])"; done
