# weight gradients in the single-CTA family (A/B): correctness vs pair, isolated, in the step
MB_WGRAD_CTA1=1 timeout 300 python -m pytest tests/test_gemm_gpu.py -q -x -k "wgrad" -p no:cacheprovider > gpurun_out/e23_gemm.log 2>&1; echo gemm=$?
for v in pair cta1; do
  e=X=1; [ $v = cta1 ] && e=MB_WGRAD_CTA1=1
  env $e timeout 120 python tools/bench_gemm.py --zipf-rows --only wgrad2 --iters 10 > gpurun_out/e23_zipf_$v.json 2>&1
  env $e timeout 120 python tools/bench_gemm.py --groups 16 --rows-per-group 4096 --only wgrad2 --iters 10 > gpurun_out/e23_g16_$v.json 2>&1
done
for v in cta1 pair cta1 pair; do
  e=X=1; [ $v = cta1 ] && e=MB_WGRAD_CTA1=1
  env $e timeout 300 python bench.py --policies relibra --batches 1 --repeats 3 --no-cpu-baseline > gpurun_out/e23_$v.json 2>> gpurun_out/e23_bench.err
  python -c "import json;d=json.loads(open('gpurun_out/e23_$v.json').read().strip().splitlines()[-1]);print('$v', round(d['ms_per_step'],3), d['roofline']['frac'], {k: v['ms'] for k, v in d['roofline']['per_kind'].items()})"
done
