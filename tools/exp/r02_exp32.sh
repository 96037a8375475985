# weight-gradient groups longest-K first (MB_WGRAD_LPT=1) vs expert order: tests, N=1, N=4
timeout 900 python -m pytest tests/test_layer_gpu.py tests/test_multirank_gpu.py -q -x -p no:cacheprovider > gpurun_out/e32_tests.log 2>&1; echo tests=$?; tail -1 gpurun_out/e32_tests.log
CUDA_VISIBLE_DEVICES=0 bash tools/ab_env.sh 1 "MB_WGRAD_LPT=1" "MB_WGRAD_LPT=0" 3
bash tools/ab_env.sh 4 "MB_WGRAD_LPT=1" "MB_WGRAD_LPT=0" 2
