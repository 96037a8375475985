# 4-GPU box: default bench at N=4 (interleaved policies + shifting-batch sequence with migration),
# then the EP=8 path (2 groups of 4) as 8 ranks on 4 GPUs (MB_OVERSUBSCRIBE=1: correctness of the
# N=8 code path and the JSON schema; timings of this mode mean nothing)
timeout 1200 python bench.py --gpus 4 > gpurun_out/e7_n4.json 2> gpurun_out/e7_n4.err; echo n4=$?
MB_OVERSUBSCRIBE=1 timeout 1500 python bench.py --gpus 8 --steps 2 --warmup 3 --repeats 1 --batches 2 --batch-steps 1 --check > gpurun_out/e7_n8_oversub.json 2> gpurun_out/e7_n8_oversub.err; echo n8=$?
