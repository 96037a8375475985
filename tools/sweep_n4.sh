# skew sweep on 4 GPUs (one process per GPU); one JSON line per run into gpurun_out/
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
P=29600
for z in 1.0 0.5 1.5 2.0; do
  P=$((P+1)); timeout 600 $TR --master-port $P bench.py --gpus 4 --zipf $z --steps 6 > gpurun_out/sw4_z$z.json 2> gpurun_out/sw4_z$z.err; echo z=$z rc=$?
done
P=$((P+1)); timeout 600 $TR --master-port $P bench.py --gpus 4 --group 2 --steps 6 > gpurun_out/sw4_g2.json 2> gpurun_out/sw4_g2.err; echo g2 rc=$?
P=$((P+1)); timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port $P bench.py --gpus 2 --steps 6 > gpurun_out/sw2_z1.0.json 2> gpurun_out/sw2_z1.0.err; echo n2 rc=$?
