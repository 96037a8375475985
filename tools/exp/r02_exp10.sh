# two-problem wgrad launch: correctness + N=1 A/B
timeout 300 python -m pytest tests/test_gemm_gpu.py -q -x -p no:cacheprovider > gpurun_out/e10_gemm.log 2>&1; echo gemm=$?
timeout 600 python -m pytest tests/test_layer_gpu.py -q -x -p no:cacheprovider > gpurun_out/e10_layer.log 2>&1; echo layer=$?
run() { name=$1; shift; env "$@" timeout 300 python bench.py --policies relibra --batches 1 --repeats 3 --no-cpu-baseline > gpurun_out/e10_$name.json 2> gpurun_out/e10_$name.err; echo $name=$?; }
run merged X=1
run split MB_WGRAD_MERGED=0
run merged_b X=1
