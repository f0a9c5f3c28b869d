mkdir -p gpurun_out
export PYTHONPATH=$PWD
timeout 600 python tools/c3_trace.py c3 5 6 2>&1 | grep -v -i warn | head -22
timeout 600 python tools/c3_trace.py c3 5 150 2>&1 | grep -v -i warn | head -22
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active --format=csv
