# Round-2 closing evidence (gpurun, one GPU): GPU tests, smoke, bench lines for every config (c4 default with the
# CPU baseline, the reference arm, c1 / c2 as CUDA-graph replays and eager, c3, c5), the c4 launch list, per-kernel
# DRAM traffic of one c4 step, and --set full captures of the rotation GEMM, the projection, the stencil and the
# digit split; each ncu leg under its own timeout and only after the same command ran clean without ncu.
mkdir -p gpurun_out
export PYTHONPATH=$PWD
P=gpurun_out/h
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
timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,lts__t_sector_hit_rate.pct \
    --clock-control none -k regex:"gemm_tn_sym_kernel|stencil5_kernel|oz_gemm_kernel|oz_slice_rows_kernel|finalize_rows_kernel" \
    -c 40 --csv $S > ${P}_c4_metrics.csv 2> ${P}_ncu_metrics.err; echo "metrics rc=$?"
timeout 600 ncu --set full --import-source on --clock-control none -k regex:oz_gemm_kernel -c 1 -f -o ${P}_oz_gemm \
  python tools/oz_bench.py 1048576 400 1 > ${P}_ncu_oz.log 2>&1; echo "oz full rc=$?"
timeout 600 ncu --set full --import-source on --clock-control none -k regex:oz_slice_rows_kernel -c 1 -f -o ${P}_oz_split \
  python tools/oz_bench.py 1048576 400 1 > ${P}_ncu_split.log 2>&1; echo "split full rc=$?"
S2="python bench.py --profile-steps 1 --dims 256,256,64"
$S2 > ${P}_plain_slab.log 2>&1 && \
timeout 600 ncu --set full --import-source on --clock-control none -k regex:stencil5_kernel -c 1 -f -o ${P}_stencil $S2 > ${P}_ncu_st.log 2>&1; echo "stencil full rc=$?"
timeout 600 ncu --set full --import-source on --clock-control none -k regex:gemm_tn_sym_kernel -s 2 -c 1 -f -o ${P}_tn_sym $S2 > ${P}_ncu_tn.log 2>&1; echo "tn full rc=$?"
tail -2 ${P}_gpu_tests.log; cat ${P}_smoke.log
for f in bench_c4 bench_c1_graph bench_c2_graph bench_c1_eager bench_c2_eager bench_c3 bench_c5; do
python -c "import json;d=json.load(open('${P}_$f.json'));print('$f',round(d['ms_per_step'],3),d['value'],d['clocks']['sm_mhz'],(d.get('cpu_baseline') or {}).get('value'), d['e2e']['value'] if d.get('e2e') else None)"; done
cat ${P}_bench_ref.json
