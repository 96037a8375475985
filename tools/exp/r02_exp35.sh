# 4 epilogue warps (two passes each) instead of 8: isolated K4 modes at the EP=1 rows
for L in libmb_sm100.so libmb_sm100_epi4.so libmb_sm100.so libmb_sm100_epi4.so; do
echo $L
MB_KERNELS_LIB=$L timeout 300 python tools/bench_gemm.py --zipf-rows --only dgrad_gated_noact,wgrad2 2>&1 | tail -1
MB_KERNELS_LIB=$L timeout 300 python tools/bench_gemm.py --zipf-rows --single --only fwd1_pregated,fwd2_store,dgrad_dx 2>&1 | tail -1
done
