# A/B of the rotation GEMM's epilogue (two-wait OZ_EPI2 vs four-wait), with
# OZ_PROF role timings (gpurun, one GPU)
mkdir -p gpurun_out
export PYTHONPATH=$PWD
for v in default variants/oz_epi1.so; do
  if [ $v = default ]; then unset SWB_LIB; else export SWB_LIB=$v; fi
  echo "== $v"; timeout 300 python tools/oz_bench.py 4194304 400 5
done > gpurun_out/epi_ab.log 2>&1
for v in variants/oz_prof.so variants/oz_prof_epi1.so; do
  echo "== $v"; SWB_LIB=$v SWB_OZ_PROF=1 timeout 300 python tools/oz_bench.py 1048576 400 1
done > gpurun_out/epi_prof.log 2>&1
unset SWB_LIB
timeout 600 python -m pytest tests/test_gpu_ozaki.py -q -x > gpurun_out/epi_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/epi_tests.log
timeout 900 python bench.py --no-cpu > gpurun_out/epi_bench_c4.json 2> gpurun_out/epi_bench_c4.err
cat gpurun_out/epi_ab.log gpurun_out/epi_prof.log; tail -2 gpurun_out/epi_tests.log
python -c "import json;d=json.load(open('gpurun_out/epi_bench_c4.json'));print(d['ms_per_step'],d['kernels']['rotation_int8_gemm'],d['clocks'])"
