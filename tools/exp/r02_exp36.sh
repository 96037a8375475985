# 4 epilogue warps vs 8 in the step: N=1 and N=4 interleaved A/B
CUDA_VISIBLE_DEVICES=0 bash tools/ab_env.sh 1 "MB_KERNELS_LIB=libmb_sm100_epi4.so" "MB_KERNELS_LIB=libmb_sm100.so" 3
bash tools/ab_env.sh 4 "MB_KERNELS_LIB=libmb_sm100_epi4.so" "MB_KERNELS_LIB=libmb_sm100.so" 2
