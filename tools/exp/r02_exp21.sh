# gated dAct in the single-CTA kernel too (A/B), N=1 and N=4
for v in d1 d0 d1 d0; do
  e=X=1; [ $v = d1 ] && e=MB_CTA1_DACT=1
  env $e timeout 300 python bench.py --policies relibra --batches 1 --repeats 3 --no-cpu-baseline > gpurun_out/e21_$v.json 2>> gpurun_out/e21_bench.err
  python -c "import json;d=json.loads(open('gpurun_out/e21_$v.json').read().strip().splitlines()[-1]);print('n1 $v', round(d['ms_per_step'],3), d['roofline']['frac'], {k: v['ms'] for k, v in d['roofline']['per_kind'].items()})"
done
for v in d1 d0; do
  e=X=1; [ $v = d1 ] && e=MB_CTA1_DACT=1
  env $e timeout 900 python bench.py --gpus 4 --policies relibra,static --batches 1 --repeats 3 > gpurun_out/e21_n4_$v.json 2>> gpurun_out/e21_bench.err
  python -c "import json;d=json.loads(open('gpurun_out/e21_n4_$v.json').read().strip().splitlines()[-1]);print('n4 $v', round(d['ms_per_step'],3), d['roofline']['frac'], d['balance']['static']['ms_per_step'], {k: v['ms'] for k, v in d['roofline']['per_kind'].items()})"
done
