mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_ozaki.py tests/test_gpu_bench_configs.py -q -x > gpurun_out/wide_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/wide_tests.log
timeout 300 python tools/oz_bench.py 4194304 400 5 > gpurun_out/wide_oz.log 2>&1
SWB_LIB=variants/oz_narrow.so timeout 300 python tools/oz_bench.py 4194304 400 5 > gpurun_out/narrow_oz.log 2>&1
timeout 900 python bench.py --no-cpu > gpurun_out/wide_bench_c4.json 2> gpurun_out/wide_bench_c4.err
tail -3 gpurun_out/wide_tests.log; cat gpurun_out/wide_oz.log gpurun_out/narrow_oz.log
python -c "import json;d=json.load(open('gpurun_out/wide_bench_c4.json'));print(d['ms_per_step'],d['roofline']['frac'],d['kernels']['rotation_int8_gemm'],d['clocks'])"
