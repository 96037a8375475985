# replay the reference-generated Qwen3 trace through the kernels on 4 GPUs: the reference's own
# plan files (--plans) and this package's planner on the same trace
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
T=tests/golden/io/qwen3_ep4
timeout 600 $TR --master-port 29961 bench.py --gpus 4 --trace $T/trace --plans $T/plans --policies relibra,static,eplb_like --steps 8 > gpurun_out/replay_plans.json 2> gpurun_out/replay_plans.err; echo plans=$?
timeout 600 $TR --master-port 29962 bench.py --gpus 4 --trace $T/trace --policies relibra,static --steps 8 > gpurun_out/replay_ours.json 2> gpurun_out/replay_ours.err; echo ours=$?
