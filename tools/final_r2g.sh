# Round-2 closing evidence, second pass (after the panel-warp seed system and the narrow / seven-segment digit split):
# GPU tests, smoke, every bench line, the reference arm, the c4 launch list and a --set full capture of the split.
mkdir -p gpurun_out
export PYTHONPATH=$PWD
P=gpurun_out/i
timeout 1500 python -m pytest tests -m gpu -x -q > ${P}_gpu_tests.log 2>&1; echo "tests rc=$?" >> ${P}_gpu_tests.log
python -c "import __graft_entry__ as g; g.smoke()" > ${P}_smoke.log 2>&1; echo "smoke rc=$?" >> ${P}_smoke.log
timeout 1200 python bench.py > ${P}_bench_c4.json 2> ${P}_bench_c4.err
timeout 900 python bench.py --impl reference --steps 2 --warmup 3 > ${P}_bench_ref.json 2> ${P}_bench_ref.err
timeout 900 python bench.py --config c1 --graph > ${P}_bench_c1_graph.json 2> ${P}_bench_c1g.err
timeout 900 python bench.py --config c2 --graph > ${P}_bench_c2_graph.json 2> ${P}_bench_c2g.err
timeout 900 python bench.py --config c1 --no-cpu > ${P}_bench_c1_eager.json 2> ${P}_bench_c1.err
timeout 900 python bench.py --config c2 --no-cpu > ${P}_bench_c2_eager.json 2> ${P}_bench_c2.err
timeout 900 python bench.py --config c3 > ${P}_bench_c3.json 2> ${P}_bench_c3.err
timeout 900 python bench.py --config c5 > ${P}_bench_c5.json 2> ${P}_bench_c5.err
S="python bench.py --profile-steps 1"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv $S > ${P}_launches_c4.csv 2> ${P}_ncu_launch.err; echo "launch list rc=$?"
timeout 600 ncu --set full --import-source on --clock-control none -k regex:oz_slice_rows_kernel -c 1 -f -o ${P}_oz_split \
  python tools/oz_bench.py 1048576 400 1 > ${P}_ncu_split.log 2>&1; echo "split full rc=$?"
tail -2 ${P}_gpu_tests.log; cat ${P}_smoke.log
for f in bench_c4 bench_c1_graph bench_c2_graph bench_c1_eager bench_c2_eager bench_c3 bench_c5; do
python -c "import json;d=json.load(open('${P}_$f.json'));print('$f',round(d['ms_per_step'],3),d['value'],d['clocks']['sm_mhz'],(d.get('cpu_baseline') or {}).get('value'), d['e2e']['value'] if d.get('e2e') else None)"; done
cat ${P}_bench_ref.json
