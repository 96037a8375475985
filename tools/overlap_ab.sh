timeout 300 python -m pytest tests/test_layer_gpu.py -x -q 2>&1 | tail -1
for i in 1 2; do for v in 1 0; do
MB_OVERLAP=$v python bench.py --no-cpu-baseline --policies relibra,balanced_oracle --steps 8 2>/dev/null | python -c "
import json,sys;d=json.loads(sys.stdin.read().strip().splitlines()[-1]);print('overlap=$v', round(d['ms_per_step'],3), round(d['balance']['balanced_oracle']['ms_per_step'],3), round(d['roofline']['gemm_ms_per_step'],3), round(d['e2e']['ms_per_step'],3), {k:v['ms'] for k,v in d['comm'].items()}, d['clocks']['sm_mhz'])"
done; done
