# dSwiGLU epilogue with double-buffered H chunks (5 stages) vs the previous (single-buffered, 6 stages)
timeout 300 python -m pytest tests/test_gemm_gpu.py -q -x -p no:cacheprovider > gpurun_out/e15_gemm.log 2>&1; echo gemm=$?
timeout 600 python -m pytest tests/test_layer_gpu.py -q -x -p no:cacheprovider > gpurun_out/e15_layer.log 2>&1; echo layer=$?
for v in new prev; do
  lib=libmb_sm100_$v.so; [ $v = new ] && lib=libmb_sm100.so
  MB_KERNELS_LIB=$lib timeout 120 python tools/bench_gemm.py --zipf-rows --only dgrad_gated --iters 30 > gpurun_out/e15_zipf_$v.json 2>&1
  MB_KERNELS_LIB=$lib timeout 120 python tools/bench_gemm.py --groups 16 --rows-per-group 4096 --only dgrad_gated --iters 30 > gpurun_out/e15_g16_$v.json 2>&1
done
for v in new prev new prev; do
  lib=libmb_sm100_$v.so; [ $v = new ] && lib=libmb_sm100.so
  MB_KERNELS_LIB=$lib timeout 300 python bench.py --policies relibra --batches 1 --repeats 3 --no-cpu-baseline > gpurun_out/e15_bench_$v.json 2>> gpurun_out/e15_bench.err
  python -c "import json;d=json.loads(open('gpurun_out/e15_bench_$v.json').read().strip().splitlines()[-1]);print('$v', round(d['ms_per_step'],3), d['roofline']['per_kind'].get('dgrad_act_gated'))"
done
