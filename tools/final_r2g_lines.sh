# Refresh the closing bench lines with the final tree (gpurun, one GPU).
mkdir -p gpurun_out
export PYTHONPATH=$PWD
P=gpurun_out/m
timeout 1200 python bench.py > ${P}_bench_c4.json 2> ${P}_bench_c4.err
timeout 900 python bench.py --impl reference --steps 2 --warmup 3 > ${P}_bench_reference.json 2> ${P}_bench_ref.err
timeout 900 python bench.py --config c1 --graph > ${P}_bench_c1_graph.json 2> ${P}_c1g.err
timeout 900 python bench.py --config c2 --graph > ${P}_bench_c2_graph.json 2> ${P}_c2g.err
timeout 900 python bench.py --config c1 --no-cpu > ${P}_bench_c1_eager.json 2> ${P}_c1.err
timeout 900 python bench.py --config c2 --no-cpu > ${P}_bench_c2_eager.json 2> ${P}_c2.err
timeout 900 python bench.py --config c3 > ${P}_bench_c3.json 2> ${P}_c3.err
timeout 900 python bench.py --config c5 > ${P}_bench_c5.json 2> ${P}_c5.err
for f in bench_c4 bench_c1_graph bench_c2_graph bench_c1_eager bench_c2_eager bench_c3 bench_c5; do
python -c "import json;d=json.load(open('${P}_$f.json'));print('$f',round(d['ms_per_step'],3),d['value'],d['clocks']['sm_mhz'],(d.get('cpu_baseline') or {}).get('value'), d['e2e']['value'] if d.get('e2e') else None)"; done
python -c "import json;d=json.load(open('${P}_bench_reference.json'));print('ref',d['value'],d['cpu_baseline']['cores'])"
