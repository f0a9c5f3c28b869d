# A/B of an environment knob on the c4 step: bash tools/gpu_ab_env.sh VAR=a VAR=b ...
export PYTHONPATH=$PWD
for v in "$@" "$@" "$@"; do
  env $v timeout 600 python bench.py --no-cpu --no-e2e --steps 6 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read()); p=d['phases_ms']
print('$v', round(d['ms_per_step'],2), d['clocks']['sm_mhz'], 'stencil', round(p['stencil'],2), 'project', round(p['project'],2), 'gemm', round(p['rotate_gemm'],2), 'join', round(p['rotate_join'],2))"
done
