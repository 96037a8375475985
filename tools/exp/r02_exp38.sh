timeout 1200 python -m pytest tests/test_layer_gpu.py -q -x -p no:cacheprovider > gpurun_out/e38_tests.log 2>&1; echo tests=$?; tail -3 gpurun_out/e38_tests.log
