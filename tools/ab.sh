# interleaved A/B of an env toggle on one box: ab.sh VAR valA valB [bench args...]
V=$1; A=$2; B=$3; shift 3
for i in 1 2 3; do
  for val in $A $B; do
    env $V=$val python bench.py --no-cpu-baseline --policies relibra --steps 8 "$@" > gpurun_out/ab_$val_$i.json 2>/dev/null
    python -c "
import json;d=json.loads(open('gpurun_out/ab_$val_$i.json').read().strip().splitlines()[-1])
print('$V=$val', round(d['ms_per_step'],3), {k:v['ms'] for k,v in d['roofline']['per_kind'].items()}, d['clocks']['sm_mhz'])"
  done
done
