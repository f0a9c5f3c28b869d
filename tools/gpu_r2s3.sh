# Round-2 session-3 check: GPU tests, smoke, c4 bench, c1 graph replay, c3.
mkdir -p gpurun_out
export PYTHONPATH=$PWD
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/s3_gpu_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/s3_gpu_tests.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/s3_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/s3_smoke.log
timeout 900 python bench.py --no-cpu > gpurun_out/s3_bench_c4.json 2> gpurun_out/s3_bench_c4.err
timeout 600 python bench.py --config c1 --graph > gpurun_out/s3_bench_c1_graph.json 2> gpurun_out/s3_bench_c1.err
timeout 600 python bench.py --config c3 > gpurun_out/s3_bench_c3.json 2> gpurun_out/s3_bench_c3.err
tail -3 gpurun_out/s3_gpu_tests.log; cat gpurun_out/s3_smoke.log
for f in s3_bench_c4 s3_bench_c1_graph s3_bench_c3; do
python -c "import json;d=json.load(open('gpurun_out/$f.json'));p=d.get('phases_ms',{});print('$f',round(d['ms_per_step'],3),d['value'],d['clocks']['sm_mhz'],{k:round(v,2) for k,v in p.items()})"; done
