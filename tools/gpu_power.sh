export PYTHONPATH=$PWD
echo "== occ default"; timeout 300 python tools/tn_power.py 16
echo "== occ 2"; SWB_TN_OCC=2 timeout 300 python tools/tn_power.py 16
echo "== occ 2, tn_bench"; SWB_TN_OCC=2 timeout 300 python tools/tn_bench.py
