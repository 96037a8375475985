# non-gated F-mode GEMMs in the single-CTA kernel: correctness + N=1 A/B
timeout 300 python -m pytest tests/test_gemm_gpu.py -q -x -p no:cacheprovider > gpurun_out/e20_gemm.log 2>&1; echo gemm=$?
timeout 600 python -m pytest tests/test_layer_gpu.py -q -x -p no:cacheprovider > gpurun_out/e20_layer.log 2>&1; echo layer=$?
for v in cta1 pair cta1 pair; do
  e=X=1; [ $v = pair ] && e=MB_CTA1_F=0
  env $e timeout 300 python bench.py --policies relibra --batches 1 --repeats 3 --no-cpu-baseline > gpurun_out/e20_$v.json 2>> gpurun_out/e20_bench.err
  python -c "import json;d=json.loads(open('gpurun_out/e20_$v.json').read().strip().splitlines()[-1]);print('$v', round(d['ms_per_step'],3), d['roofline']['frac'], {k: v['ms'] for k, v in d['roofline']['per_kind'].items()})"
done
