timeout 300 python -m pytest tests/test_layer_gpu.py -x -q 2>&1 | tail -1
for i in 1 2; do python bench.py --no-cpu-baseline --policies relibra --steps 8 2>/dev/null | python -c "
import json,sys;d=json.loads(sys.stdin.read().strip().splitlines()[-1]);print('n1', round(d['ms_per_step'],3), 'e2e', round(d['e2e']['ms_per_step'],3), d['clocks']['sm_mhz'])"; done
