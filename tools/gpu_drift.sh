mkdir -p gpurun_out
export PYTHONPATH=$PWD
timeout 600 python tools/step_drift.py c3 150 2>&1 | grep -v Warn | cut -c1-110
timeout 600 python bench.py --config c3 --no-cpu > gpurun_out/c3_base.json 2> gpurun_out/c3_base.err
python -c "import json;d=json.load(open('gpurun_out/c3_base.json'));print(d['ms_per_step'],d['steps'],d['clocks'],d['e2e'])"
