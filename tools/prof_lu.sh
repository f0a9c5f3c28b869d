# seed-system LU pieces (c4 seeds: S = 800 -> 801 x 801) -- one --set full capture of a panel and of getrs
S="python bench.py --profile-steps 1 --dims 128,128,128"
$S > gpurun_out/plain_lu.log 2>&1 && \
ncu --set full --import-source on --clock-control none -k regex:"panel_kernel|getrs_kernel" -s 2 -c 2 -f -o gpurun_out/lu_full $S \
    > gpurun_out/ncu_lu.log 2>&1
echo rc=$?
