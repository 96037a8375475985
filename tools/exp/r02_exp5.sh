# K4: 6 operand stages + 32-feature dSwiGLU chunks vs round 1 (r1) and 5 stages (s5)
timeout 600 python -m pytest tests/test_gemm_gpu.py tests/test_layer_gpu.py -q -x -p no:cacheprovider > gpurun_out/e5_pytest.log 2>&1; echo pytest=$?
for v in r1 s5 new; do
  lib=libmb_sm100_$v.so; [ $v = new ] && lib=libmb_sm100.so
  MB_KERNELS_LIB=$lib python tools/bench_gemm.py --zipf-rows --only fwd1_swiglu,fwd2_store,dgrad_gated,dgrad_dx --iters 30 > gpurun_out/e5_zipf_$v.json 2>&1
  MB_KERNELS_LIB=$lib python tools/bench_gemm.py --groups 16 --rows-per-group 4096 --only fwd1_swiglu,fwd2_store,dgrad_gated,dgrad_dx,wgrad_w1,wgrad_w2 --iters 30 > gpurun_out/e5_g16_$v.json 2>&1
done
for v in r1prof prof; do
  for m in fwd1_swiglu dgrad_gated dgrad_dx; do
    MB_KERNELS_LIB=libmb_sm100_$v.so MB_GEMM_PROF=1 python tools/bench_gemm.py --zipf-rows --only $m --iters 2 --warmup 1 > gpurun_out/e5_prof_${v}_$m.log 2>&1
  done
done
for v in r1 new; do
  lib=libmb_sm100_$v.so; [ $v = new ] && lib=libmb_sm100.so
  MB_KERNELS_LIB=$lib timeout 600 python bench.py --policies relibra --batches 1 --repeats 3 --no-cpu-baseline > gpurun_out/e5_bench_$v.json 2> gpurun_out/e5_bench_$v.err
done
