mkdir -p gpurun_out
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
timeout 300 $TR --master-port 29511 tools/mgpu_check.py --config tiny --micro-batches 3 --steps 2 > gpurun_out/m4_tiny.log 2>&1; echo tiny=$?
timeout 300 $TR --master-port 29512 tools/mgpu_check.py --config qwen3-30b-a3b --tokens 2048 --micro-batches 3 --group 2 --steps 2 > gpurun_out/m4_q_g2.log 2>&1; echo qg2=$?
timeout 300 $TR --master-port 29513 tools/mgpu_check.py --config qwen3-30b-a3b --tokens 2048 --micro-batches 4 --steps 2 > gpurun_out/m4_q_g4.log 2>&1; echo qg4=$?
timeout 600 $TR --master-port 29514 bench.py --gpus 4 > gpurun_out/b4s.json 2> gpurun_out/b4s.err; echo b4=$?
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29515 bench.py --gpus 2 > gpurun_out/b2s.json 2> gpurun_out/b2s.err; echo b2=$?
