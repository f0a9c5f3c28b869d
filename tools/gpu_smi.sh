mkdir -p gpurun_out
export PYTHONPATH=$PWD
for ms in 200 2000 50; do
SWB_SMI_MS=$ms timeout 600 python bench.py --config c3 --no-cpu --no-e2e > gpurun_out/smi_c3_$ms.json 2>/dev/null
python -c "import json;d=json.load(open('gpurun_out/smi_c3_$ms.json'));print('c3 smi $ms', round(d['ms_per_step'],3), d['steps'], d['clocks'])"
done
SWB_SMI_MS=2000 timeout 600 python bench.py --config c1 --no-cpu --no-e2e > gpurun_out/smi_c1.json 2>/dev/null
python -c "import json;d=json.load(open('gpurun_out/smi_c1.json'));print('c1 eager smi 2000', round(d['ms_per_step'],3), d['steps'])"
timeout 600 python bench.py --config c1 --no-cpu --no-e2e > gpurun_out/smi_c1b.json 2>/dev/null
python -c "import json;d=json.load(open('gpurun_out/smi_c1b.json'));print('c1 eager smi 200', round(d['ms_per_step'],3), d['steps'])"
