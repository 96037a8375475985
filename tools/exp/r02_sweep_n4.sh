# skew / fluctuation sweep and the other BASELINE shapes at N=4 (and N=2), current code
B="python bench.py --batches 1"
for z in 0.5 1.5 2.0; do
  timeout 900 $B --gpus 4 --zipf $z --no-cpu-baseline > gpurun_out/s4_z$z.json 2> gpurun_out/s4_z$z.err; echo n4_z$z=$?
done
timeout 900 $B --gpus 4 --hot-shift 32 > gpurun_out/s4_shift32.json 2> gpurun_out/s4_shift32.err; echo n4_shift32=$?
timeout 900 $B --gpus 2 --zipf 1.5 > gpurun_out/s2_z1.5.json 2> gpurun_out/s2_z1.5.err; echo n2_z1.5=$?
timeout 1200 $B --gpus 4 --config mixtral-8x7b --repeats 2 > gpurun_out/s4_mixtral.json 2> gpurun_out/s4_mixtral.err; echo mixtral=$?
timeout 1200 $B --gpus 4 --config qwen3-235b-a22b --group 2 --repeats 2 > gpurun_out/s4_235b.json 2> gpurun_out/s4_235b.err; echo q235=$?
