# dSwiGLU epilogue in 64-feature segments with 128-byte rows (libmb_sm100_wide.so, 5 operand stages)
MB_KERNELS_LIB=libmb_sm100_wide.so timeout 600 python -m pytest tests/test_gemm_gpu.py -q -x -p no:cacheprovider > gpurun_out/e34_tests.log 2>&1; echo tests=$?; tail -1 gpurun_out/e34_tests.log
for i in 1 2; do for L in libmb_sm100.so libmb_sm100_wide.so; do
echo $L; MB_KERNELS_LIB=$L timeout 300 python tools/bench_gemm.py --zipf-rows --only dgrad_gated_noact,dgrad_gated 2>&1 | tail -1
MB_KERNELS_LIB=$L timeout 300 python tools/bench_gemm.py --groups 16 --rows-per-group 4096 --only dgrad_gated_noact 2>&1 | tail -1
done; done
bash tools/ab_env.sh 1 "MB_KERNELS_LIB=libmb_sm100.so" "MB_KERNELS_LIB=libmb_sm100_wide.so" 3
