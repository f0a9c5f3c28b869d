# stencil pass at c4 line geometry (256 x 256 x 64, K = 400): one --set full capture
S="python bench.py --profile-steps 1 --dims 256,256,64"
$S > gpurun_out/plain_st.log 2>&1 && \
ncu --set full --import-source on --clock-control none -k regex:stencil[56] -c 1 -f -o gpurun_out/st_full $S \
    > gpurun_out/ncu_st.log 2>&1
echo rc=$?
