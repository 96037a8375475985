# skew sweep at N=2 (Zipf s; every policy): gpurun_out/sw2_z*.json
for z in 0.5 1.0 1.5 2.0; do
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 2987${z%.*} bench.py --gpus 2 --zipf $z --steps 6 --no-cpu-baseline > gpurun_out/sw2_z$z.json 2>/dev/null; echo z$z=$?
done
