python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29701 bench.py --gpus 4 --steps 6 --policies relibra,balanced_oracle > gpurun_out/n4c.json 2> gpurun_out/n4c.err; echo rc=$?
python bench.py --steps 6 --policies relibra --no-cpu-baseline > gpurun_out/n1c.json 2> gpurun_out/n1c.err; echo rc=$?
