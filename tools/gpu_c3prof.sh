# c3 step: kernel launch list over 5 steps (one per interaction round)
mkdir -p gpurun_out
export PYTHONPATH=$PWD
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv python bench.py --config c3 --profile-steps 10 > gpurun_out/c3_ncu.csv 2> gpurun_out/c3_ncu.err
echo rc=$?
