# light epilogues: double-buffered output boxes with 5 operand stages (lb2) vs one box, 6 stages
timeout 300 env MB_KERNELS_LIB=libmb_sm100_lb2.so python -m pytest tests/test_gemm_gpu.py -q -x -p no:cacheprovider > gpurun_out/e17_gemm.log 2>&1; echo gemm=$?
for v in new lb2; do
  lib=libmb_sm100_$v.so; [ $v = new ] && lib=libmb_sm100.so
  MB_KERNELS_LIB=$lib timeout 120 python tools/bench_gemm.py --zipf-rows --only fwd1_swiglu,fwd2_store,dgrad_dx --iters 30 > gpurun_out/e17_zipf_$v.json 2>&1
  MB_KERNELS_LIB=$lib timeout 120 python tools/bench_gemm.py --groups 16 --rows-per-group 4096 --only fwd1_swiglu,fwd2_store,dgrad_dx,wgrad2 --iters 30 > gpurun_out/e17_g16_$v.json 2>&1
done
for v in new lb2 new lb2; do
  lib=libmb_sm100_$v.so; [ $v = new ] && lib=libmb_sm100.so
  MB_KERNELS_LIB=$lib timeout 300 python bench.py --policies relibra --batches 1 --repeats 3 --no-cpu-baseline > gpurun_out/e17_bench_$v.json 2>> gpurun_out/e17_bench.err
  python -c "import json;d=json.loads(open('gpurun_out/e17_bench_$v.json').read().strip().splitlines()[-1]);print('$v', round(d['ms_per_step'],3), d['roofline']['frac'], {k: v['ms'] for k, v in d['roofline']['per_kind'].items()})"
done
