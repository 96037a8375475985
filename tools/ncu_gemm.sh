# one ncu --set full capture per GEMM mode (pair kernel), balanced rows; run on ONE GPU
for m in fwd1_swiglu dgrad_gated dgrad_dx wgrad_w1; do
  ncu --set full --clock-control none --import-source on -k regex:grouped_gemm -s 3 -c 1 \
      -o gpurun_out/r01_$m -f python tools/bench_gemm.py --only $m --iters 1 --warmup 3 > gpurun_out/ncu_$m.log 2>&1
done
