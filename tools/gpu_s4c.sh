# c1 eager launch list (one step after warm-up) to see the dependent-kernel chain
mkdir -p gpurun_out
export PYTHONPATH=$PWD
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv python bench.py --config c1 --profile-steps 3 \
  > gpurun_out/s4c_launches_c1.csv 2> gpurun_out/s4c_ncu.err; echo "rc=$?"
wc -l gpurun_out/s4c_launches_c1.csv
