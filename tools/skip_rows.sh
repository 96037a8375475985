for i in 1 2; do for v in 0 1; do
MB_PROFILE_SKIP_ROWS=$v python bench.py --no-cpu-baseline --policies relibra --steps 8 2>/dev/null | python -c "
import json,sys;d=json.loads(sys.stdin.read().strip().splitlines()[-1]);print('skip=$v', round(d['ms_per_step'],3), round(d['roofline']['gemm_ms_per_step'],3), {k:v['ms'] for k,v in d['roofline']['per_kind'].items()}, d['clocks']['sm_mhz'])"
done; done
