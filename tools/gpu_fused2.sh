mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_update_and_solve.py -q -x > gpurun_out/fused_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/fused_tests.log
timeout 600 python bench.py --config c1 --no-cpu > gpurun_out/fused_bench_c1.json 2> gpurun_out/fused_bench_c1.err
timeout 600 python bench.py --config c2 --no-cpu > gpurun_out/fused_bench_c2.json 2>> gpurun_out/fused_bench_c1.err
tail -15 gpurun_out/fused_tests.log; tail -3 gpurun_out/fused_bench_c1.err
for f in fused_bench_c1 fused_bench_c2; do
python -c "import json;d=json.load(open('gpurun_out/$f.json'));print('$f',d['ms_per_step'],d['e2e']['ms_per_step'])"; done
