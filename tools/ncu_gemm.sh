# one ncu --set full capture per GEMM mode (pair kernel); run on ONE GPU.  Shapes: the EP=8
# per-GPU shape (16 experts x 4096 rows) and one EP=1 micro-batch (128 experts x 512 rows).
for shape in "16 4096" "128 512"; do
  set -- $shape
  for m in fwd1_swiglu fwd2_store dgrad_gated dgrad_dx wgrad_w1; do
    ncu --set full --clock-control none --import-source on -k regex:grouped_gemm -s 3 -c 1 \
        -o gpurun_out/r01_${m}_g$1 -f python tools/bench_gemm.py --only $m --iters 1 --warmup 3 \
        --groups $1 --rows-per-group $2 > gpurun_out/ncu_${m}_g$1.log 2>&1
  done
done
