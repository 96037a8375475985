# skew / fluctuation sweep and the other BASELINE shapes at N=4 (and N=2), current code
B="python bench.py --batches 1"
for z in 0.5 1.5 2.0; do
  timeout 900 $B --gpus 4 --zipf $z --no-cpu-baseline > gpurun_out/s4_z$z.json 2> gpurun_out/s4_z$z.err; echo n4_z$z=$?
done
timeout 900 $B --gpus 4 --hot-shift 32 > gpurun_out/s4_shift32.json 2> gpurun_out/s4_shift32.err; echo n4_shift32=$?
timeout 900 $B --gpus 2 --zipf 1.5 > gpurun_out/s2_z1.5.json 2> gpurun_out/s2_z1.5.err; echo n2_z1.5=$?
timeout 1200 $B --gpus 4 --config mixtral-8x7b --repeats 2 > gpurun_out/s4_mixtral.json 2> gpurun_out/s4_mixtral.err; echo mixtral=$?
timeout 1200 $B --gpus 4 --config qwen3-235b-a22b --group 2 --repeats 2 > gpurun_out/s4_235b.json 2> gpurun_out/s4_235b.err; echo q235=$?
for f in s4_z0.5 s4_z1.5 s4_z2.0 s4_shift32 s2_z1.5 s4_mixtral s4_235b; do python -c "
import json;d=json.loads(open('gpurun_out/$f.json').read().strip().splitlines()[-1]);b=d['balance']
g=lambda k: round(b[k]['ms_per_step'],2) if isinstance(b.get(k),dict) else None
print('$f', g('relibra'), g('static'), g('eplb_like'), g('balanced_oracle'), round(b['speedup_vs_static'],3), round(b['model_predicted_speedup_vs_static'],3), round(b['frac_of_balanced'],3), g('relibra_box'))" 2>&1 | tail -1; done
