# last code state: default bench lines N=1 / 2 / 4 on one 4-GPU box
CUDA_VISIBLE_DEVICES=0 timeout 900 python bench.py > gpurun_out/g6_n1.json 2> gpurun_out/g6_n1.err; echo n1=$?
timeout 900 python bench.py --gpus 2 > gpurun_out/g6_n2.json 2> gpurun_out/g6_n2.err; echo n2=$?
timeout 1200 python bench.py --gpus 4 > gpurun_out/g6_n4.json 2> gpurun_out/g6_n4.err; echo n4=$?
for f in g6_n1 g6_n2 g6_n4; do python -c "
import json;d=json.loads(open('gpurun_out/$f.json').read().strip().splitlines()[-1]);b=d.get('balance',{})
g=lambda k: round(b[k]['ms_per_step'],2) if isinstance(b.get(k),dict) else None
print('$f', round(d['ms_per_step'],3), round(d['value']/1e6,3), d['roofline']['frac'], d['clocks']['sm_mhz'], round(d['e2e']['value']/1e6,3), g('relibra'), g('static'), g('eplb_like'), g('balanced_oracle'), b.get('speedup_vs_static'), b.get('frac_of_balanced'))"; done
