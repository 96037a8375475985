# interleaved A/B of an environment switch on the bench step: ab_env.sh N "ENV_A" "ENV_B" [reps]
N=$1; A=$2; B=$3; R=${4:-2}
P=29850
for i in $(seq $R); do
  for E in "$A" "$B"; do
    P=$((P+1))
    if [ "$N" = 1 ]; then cmd="python bench.py"; else cmd="python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port $P bench.py --gpus $N"; fi
    env $E timeout 600 $cmd --no-cpu-baseline --policies relibra --steps ${STEPS:-8} $BENCH_ARGS 2>/dev/null | python -c "
import json,sys;d=json.loads(sys.stdin.read().strip().splitlines()[-1]);print('$N [$E]', round(d['ms_per_step'],3), 'gemm', round(d['roofline']['gemm_ms_per_step'],2), {k:round(v['ms'],2) for k,v in d['roofline']['per_kind'].items()}, d['clocks']['sm_mhz'])"
  done
done
