# interleaved A/B of two kernel-library builds on one box: ab_lib.sh libA libB
A=$1; B=$2
O=fwd1_swiglu,fwd2_store,dgrad_gated,dgrad_dx,wgrad_w2,wgrad_w1
timeout 300 env MB_KERNELS_LIB=$B python -m pytest tests/test_gemm_gpu.py -x -q 2>&1 | tail -1
for i in 1 2; do
  for L in $A $B; do
    echo "== $L"
    MB_KERNELS_LIB=$L python tools/bench_gemm.py --only $O --groups 16 --rows-per-group 4096
    MB_KERNELS_LIB=$L python tools/bench_gemm.py --only $O --zipf-rows
    MB_KERNELS_LIB=$L python bench.py --no-cpu-baseline --policies relibra --steps 8 2>/dev/null | python -c "
import json,sys;d=json.loads(sys.stdin.read().strip().splitlines()[-1]);print('step', round(d['ms_per_step'],3), {k:v['ms'] for k,v in d['roofline']['per_kind'].items()}, d['clocks']['sm_mhz'])"
  done
done
