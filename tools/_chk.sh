timeout 600 python -m pytest tests/test_layer_gpu.py -x -q > gpurun_out/pt_l.log 2>&1; echo pytest=$?; tail -1 gpurun_out/pt_l.log
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
timeout 300 $TR --master-port 29951 tools/mgpu_check.py --config qwen3-30b-a3b --tokens 2048 --micro-batches 3 --group 2 --steps 2 > gpurun_out/c4_b.log 2>&1; echo chk=$?
timeout 300 $TR --master-port 29911 tools/step_timeline.py > gpurun_out/tl4.log 2>&1; echo tl=$?
bash tools/ab_env.sh 4 "MB_X=1" "MB_X=2" 1 > gpurun_out/ab_b4.log 2>&1
bash tools/ab_env.sh 1 "MB_X=1" "MB_X=2" 1 > gpurun_out/ab_b1.log 2>&1
