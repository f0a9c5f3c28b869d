export PYTHONPATH=$PWD
mkdir -p gpurun_out
timeout 300 python tools/tn_bench.py 1048576 400 3
echo "== interleave (default)"; timeout 300 python tools/tn_bench.py
echo "== contiguous"; SWB_TN_INTERLEAVE=0 timeout 300 python tools/tn_bench.py
timeout 300 ncu --metrics dram__bytes_read.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct --clock-control none -k regex:gemm_tn_sym -c 1 python tools/tn_bench.py 16777216 400 1 2>&1 | grep -E "dram__|gpu__time|lts__" 
SWB_TN_INTERLEAVE=0 timeout 300 ncu --metrics dram__bytes_read.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct --clock-control none -k regex:gemm_tn_sym -c 1 python tools/tn_bench.py 16777216 400 1 2>&1 | grep -E "dram__|gpu__time|lts__"
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x 2>&1 | tail -2
