export PYTHONPATH=$PWD
for v in default variants/sp_8w32r.so variants/sp_4w16r_m8.so variants/sp_4w32r.so variants/sp_2w8r.so; do
  if [ $v = default ]; then unset SWB_LIB; else export SWB_LIB=$v; fi
  echo "== $v"; timeout 120 python tools/split_bench.py 1048576 400
done
