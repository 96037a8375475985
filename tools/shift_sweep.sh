# hot-set fluctuation sweep at N=4 (experts the hot set rotates by per micro-batch), Zipf 1.0 and 1.5
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
P=29890
for z in 1.0 1.5; do for sh in 0 32 64; do P=$((P+1))
  timeout 600 $TR --master-port $P bench.py --gpus 4 --zipf $z --hot-shift $sh --steps 6 --no-cpu-baseline > gpurun_out/shift_z${z}_s$sh.json 2>/dev/null; echo z$z s$sh=$?
done; done
