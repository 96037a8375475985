# dynamic tile scheduling in the CTA-pair GEMM: correctness first (short timeouts), then A/B
timeout 300 python -m pytest tests/test_gemm_gpu.py -q -x -p no:cacheprovider > gpurun_out/e9_gemm.log 2>&1; echo gemm=$?
timeout 600 python -m pytest tests/test_layer_gpu.py -q -x -p no:cacheprovider > gpurun_out/e9_layer.log 2>&1; echo layer=$?
for v in dyn static; do
  e=X=1; [ $v = static ] && e=MB_GEMM_STATIC=1
  env $e timeout 120 python tools/bench_gemm.py --zipf-rows --iters 30 > gpurun_out/e9_zipf_$v.json 2>&1
  env $e timeout 120 python tools/bench_gemm.py --groups 16 --rows-per-group 4096 --iters 30 > gpurun_out/e9_g16_$v.json 2>&1
done
run() { name=$1; shift; env "$@" timeout 300 python bench.py --policies relibra --batches 1 --repeats 3 --no-cpu-baseline > gpurun_out/e9_$name.json 2> gpurun_out/e9_$name.err; echo $name=$?; }
run dyn0 X=1
run static0 MB_GEMM_STATIC=1
run dyn8 MB_COMM_SMS=8
run dyn20 MB_COMM_SMS=20
run dynserial MB_OVERLAP=0
