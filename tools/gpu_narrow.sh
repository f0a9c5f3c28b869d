mkdir -p gpurun_out
export PYTHONPATH=$PWD
timeout 900 python -m pytest tests/test_gpu_ozaki.py tests/test_gpu_update_and_solve.py tests/test_gpu_emit.py -q -x > gpurun_out/narrow_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/narrow_tests.log
for v in default variants/oz_nonarrow.so default variants/oz_nonarrow.so; do
  if [ $v = default ]; then unset SWB_LIB; else export SWB_LIB=$v; fi
  echo "== $v"; timeout 300 python tools/oz_bench.py 4194304 400 8 2>&1 | head -1
done > gpurun_out/narrow_oz.log
unset SWB_LIB
timeout 900 python bench.py --no-cpu > gpurun_out/narrow_bench_c4.json 2> gpurun_out/narrow_bench_c4.err
tail -3 gpurun_out/narrow_tests.log; cat gpurun_out/narrow_oz.log
python -c "import json;d=json.load(open('gpurun_out/narrow_bench_c4.json'));p=d['phases_ms'];print(round(d['ms_per_step'],1),d['clocks']['sm_mhz'],round(p['project'],2),round(p['rotate_split'],2),round(p['rotate_gemm'],2),round(p['rotate_join'],2),round(p['stencil'],2))"
