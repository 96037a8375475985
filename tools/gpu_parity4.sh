TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/pt4.log 2>&1; echo pytest=$?; tail -2 gpurun_out/pt4.log
timeout 300 $TR --master-port 29951 tools/mgpu_check.py --config qwen3-30b-a3b --tokens 2048 --micro-batches 3 --group 2 --steps 2 > gpurun_out/c4.log 2>&1; echo chk=$?
timeout 300 $TR --master-port 29952 tools/mgpu_check.py --config tiny --micro-batches 3 --steps 2 > gpurun_out/c4t.log 2>&1; echo chkt=$?
timeout 300 $TR --master-port 29953 tools/mgpu_migrate.py --config qwen3-30b-a3b --tokens 1024 > gpurun_out/m4.log 2>&1; echo mig=$?
for i in 1 2; do timeout 600 $TR --master-port $((29960+i)) bench.py --gpus 4 --steps 8 --policies relibra,balanced_oracle 2>/dev/null | python -c "
import json,sys;d=json.loads(sys.stdin.read().strip().splitlines()[-1]);print('n4', round(d['ms_per_step'],3), {k:round(v['ms_per_step'],3) for k,v in d['balance'].items() if isinstance(v,dict)}, {k:v['ms'] for k,v in d['comm'].items()}, d['clocks']['sm_mhz'])"; done
