TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
timeout 300 $TR --master-port 29911 tools/mgpu_migrate.py --config tiny > gpurun_out/mig_tiny.log 2>&1; echo tiny=$?
timeout 300 $TR --master-port 29912 tools/mgpu_migrate.py --config qwen3-30b-a3b --tokens 1024 > gpurun_out/mig_q.log 2>&1; echo q=$?
timeout 300 $TR --master-port 29913 tools/mgpu_check.py --config qwen3-30b-a3b --tokens 2048 --micro-batches 3 --group 2 --steps 2 > gpurun_out/chk_q.log 2>&1; echo chk=$?
