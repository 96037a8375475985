# EP=8 correctness with 8 ranks on a 2- or 4-GPU box (MB_OVERSUBSCRIBE=1, gloo host group, CUDA-IPC
# between the rank processes).  Timings of this mode are meaningless.
export MB_OVERSUBSCRIBE=1
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 8 --master-addr 127.0.0.1"
timeout 900 $TR --master-port 29971 tests/mgpu_worker.py --config qwen3-30b-a3b --tokens 1024 --micro-batches 2 \
    --zipf 1.5 --group 4 --migrate > gpurun_out/o8_worker.log 2>&1; echo worker=$?
timeout 1500 python bench.py --gpus 8 --steps 2 --warmup 3 --repeats 1 --batches 2 --batch-steps 1 --check \
    > gpurun_out/o8_bench.json 2> gpurun_out/o8_bench.err; echo bench=$?
