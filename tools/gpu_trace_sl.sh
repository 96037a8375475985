timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
timeout 300 $TR --master-port 29971 bench.py --gpus 4 --trace tests/golden/io/samples2/trace --plans tests/golden/io/samples2/plans_sl --policies relibra,static --steps 3 > gpurun_out/tr_sl.json 2> gpurun_out/tr_sl.err; echo sl=$?; tail -2 gpurun_out/tr_sl.err
timeout 300 $TR --master-port 29972 bench.py --gpus 4 --trace tests/golden/io/samples2/trace --plans tests/golden/io/samples2/plans --policies relibra --steps 3 > gpurun_out/tr_nosl.json 2> gpurun_out/tr_nosl.err; echo nosl=$?
