# single-CTA tail tiles: correctness, then N=1 A/B
timeout 300 python -m pytest tests/test_gemm_gpu.py -q -x -p no:cacheprovider > gpurun_out/e13_gemm.log 2>&1; echo gemm=$?
timeout 600 python -m pytest tests/test_layer_gpu.py -q -x -p no:cacheprovider > gpurun_out/e13_layer.log 2>&1; echo layer=$?
run() { name=$1; shift; env "$@" timeout 300 python bench.py --policies relibra --batches 1 --repeats 3 --no-cpu-baseline > gpurun_out/e13_$name.json 2> gpurun_out/e13_$name.err; echo $name=$?; }
run tails X=1
run notails MB_TAIL_TILES=0
run tails_b X=1
run notails_b MB_TAIL_TILES=0
