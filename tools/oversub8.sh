# EP=8 correctness on a 2-GPU box: 8 ranks, 4 per GPU (MB_OVERSUBSCRIBE=1, gloo host group,
# CUDA-IPC between ranks on the same GPU and across the pair).  Timings are meaningless here.
export MB_OVERSUBSCRIBE=1
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 8 --master-addr 127.0.0.1"
timeout 600 $TR --master-port 29971 tools/mgpu_check.py --config tiny --micro-batches 3 --steps 2 > gpurun_out/o8_tiny.log 2>&1; echo chk_tiny=$?
timeout 900 $TR --master-port 29972 tools/mgpu_check.py --config qwen3-30b-a3b --tokens 1024 --micro-batches 3 --steps 2 > gpurun_out/o8_qwen.log 2>&1; echo chk_qwen=$?
timeout 900 $TR --master-port 29973 tools/mgpu_migrate.py --config qwen3-30b-a3b --tokens 512 > gpurun_out/o8_mig.log 2>&1; echo mig=$?
timeout 1200 $TR --master-port 29974 bench.py --gpus 8 --steps 1 --warmup 1 --policies relibra,static,relibra_box --sa-chains 4 > gpurun_out/o8_bench.json 2> gpurun_out/o8_bench.err; echo bench=$?
