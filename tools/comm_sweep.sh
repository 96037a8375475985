# step time vs row-mover engine / SM split: comm_sweep.sh N "blocks:gemm_sms ..." (0:0 = register movers, default split)
N=$1; shift
P=29800
for v in $*; do
  nb=${v%%:*}; gs=${v##*:}
  P=$((P+1))
  envs="MB_COMM_BLOCKS=$nb"; [ "$gs" != 0 ] && envs="$envs MB_GEMM_SMS=$gs"
  if [ "$N" = 1 ]; then cmd="python bench.py"; else cmd="python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port $P bench.py --gpus $N"; fi
  env $envs timeout 600 $cmd --no-cpu-baseline --policies relibra --steps 8 2>gpurun_out/sweep_err_$nb_$gs.log | python -c "
import json,sys;d=json.loads(sys.stdin.read().strip().splitlines()[-1]);print('$N $v', round(d['ms_per_step'],3), 'gemm', round(d['roofline']['gemm_ms_per_step'],2), {k:round(v['ms'],2) for k,v in d['roofline']['per_kind'].items()}, 'comm', {k:round(v['ms'],2) for k,v in d['comm'].items()}, d['clocks']['sm_mhz'])"
done
