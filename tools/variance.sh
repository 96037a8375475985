# repeated bench lines (run-to-run spread on one box): N=1 x3, then N=4 x3 when 4 GPUs are visible
for i in 1 2 3; do timeout 600 python bench.py --policies relibra,static --no-cpu-baseline > gpurun_out/var_n1_$i.json 2>/dev/null; echo n1_$i=$?; done
if [ "$(nvidia-smi -L | wc -l)" -ge 4 ]; then
  for i in 1 2 3; do timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port $((29940+i)) bench.py --gpus 4 --policies relibra,static --no-cpu-baseline > gpurun_out/var_n4_$i.json 2>/dev/null; echo n4_$i=$?; done
fi
