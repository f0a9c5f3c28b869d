# rotation: conflict-free split staging, overlapped vs serial split (gpurun, one GPU)
mkdir -p gpurun_out
export PYTHONPATH=$PWD
for v in default variants/oz_serial.so; do
  if [ $v = default ]; then unset SWB_LIB; else export SWB_LIB=$v; fi
  echo "== $v"; timeout 300 python tools/oz_bench.py 4194304 400 5
done > gpurun_out/split_ab.log 2>&1
unset SWB_LIB
timeout 600 python -m pytest tests/test_gpu_ozaki.py -q -x > gpurun_out/split_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/split_tests.log
timeout 900 python bench.py --no-cpu --no-e2e > gpurun_out/split_bench_c4.json 2> gpurun_out/split_bench_c4.err
SWB_OZ_SERIAL=1 timeout 900 python bench.py --no-cpu --no-e2e > gpurun_out/split_bench_c4_serial.json 2>> gpurun_out/split_bench_c4.err
cat gpurun_out/split_ab.log; tail -2 gpurun_out/split_tests.log
for f in split_bench_c4 split_bench_c4_serial; do
python -c "import json;d=json.load(open('gpurun_out/$f.json'));print('$f',d['ms_per_step'],d['kernels']['rotation'],d['kernels']['rotation_int8_gemm']['ms'],d['clocks'])"; done
