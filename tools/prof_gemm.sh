# projection (TN sym) and rotation (NN) GEMMs at c4 row geometry (256 x 256 x 64, K = 400): --set full
S="python bench.py --profile-steps 1 --dims 256,256,64"
$S > gpurun_out/plain_gemm.log 2>&1 && \
ncu --set full --import-source on --clock-control none -k regex:"gemm_tn_sym_kernel|gemm_nn_kernel" -s 4 -c 2 -f \
    -o gpurun_out/gemm_full $S > gpurun_out/ncu_gemm.log 2>&1
echo rc=$?
