# Full GPU check of the current tree (run under gpurun): tests, smoke, bench (ours + reference arm)
mkdir -p gpurun_out
python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/gpu_tests.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
python bench.py > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err
python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
python bench.py --config c5 --no-cpu > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err
tail -3 gpurun_out/gpu_tests.log; cat gpurun_out/smoke.log gpurun_out/bench_c4.json
