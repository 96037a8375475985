TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
P=29940
for i in 1 2; do for L in libmb_sm100_w8.so libmb_sm100.so; do
P=$((P+1))
MB_KERNELS_LIB=$L timeout 600 $TR --master-port $P bench.py --gpus 4 --steps 8 --policies relibra,balanced_oracle 2>/dev/null | python -c "
import json,sys;d=json.loads(sys.stdin.read().strip().splitlines()[-1]);print('$L', round(d['ms_per_step'],3), {k:round(v['ms_per_step'],3) for k,v in d['balance'].items() if isinstance(v,dict)}, {k:v['ms'] for k,v in d['roofline']['per_kind'].items()}, {k:v['ms'] for k,v in d['comm'].items()}, d['clocks']['sm_mhz'])"
done; done
