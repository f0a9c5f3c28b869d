export PYTHONPATH=$PWD
for v in default variants/oz_st5.so variants/oz_st3.so default variants/oz_st5.so; do
  if [ $v = default ]; then unset SWB_LIB; else export SWB_LIB=$v; fi
  echo "== $v"; timeout 300 python tools/oz_bench.py 4194304 400 8 2>&1 | head -1
done
