# final N=4 / N=2 on a 4-GPU box (default bench), N=4 with --check, reference arm at N=4
timeout 1200 python bench.py --gpus 4 > gpurun_out/f4_bench.json 2> gpurun_out/f4_bench.err; echo n4=$?
timeout 900 python bench.py --gpus 2 > gpurun_out/f2_bench.json 2> gpurun_out/f2_bench.err; echo n2=$?
timeout 900 python bench.py --gpus 4 --check --batches 1 --policies relibra > gpurun_out/f4_check.json 2> gpurun_out/f4_check.err; echo n4check=$?
WORLD_SIZE=4 RANK=0 timeout 900 python bench.py --gpus 4 --impl reference --steps 3 --warmup 1 > gpurun_out/f4_ref.json 2> gpurun_out/f4_ref.err; echo ref4=$?
