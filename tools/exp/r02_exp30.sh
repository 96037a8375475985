# dSwiGLU epilogue reading H through global loads (libmb_sm100_ldg.so) vs TMA boxes (default)
MB_KERNELS_LIB=libmb_sm100_ldg.so timeout 600 python -m pytest tests/test_gemm_gpu.py -q -x -p no:cacheprovider -k "dswiglu" > gpurun_out/e30_tests.log 2>&1; echo tests=$?; tail -1 gpurun_out/e30_tests.log
for i in 1 2; do for L in libmb_sm100.so libmb_sm100_ldg.so; do
echo $L; MB_KERNELS_LIB=$L timeout 300 python tools/bench_gemm.py --zipf-rows --only dgrad_gated_noact 2>&1 | tail -1
MB_KERNELS_LIB=$L timeout 300 python tools/bench_gemm.py --groups 16 --rows-per-group 4096 --only dgrad_gated_noact 2>&1 | tail -1
done; done
bash tools/ab_env.sh 1 "MB_KERNELS_LIB=libmb_sm100.so" "MB_KERNELS_LIB=libmb_sm100_ldg.so" 3
