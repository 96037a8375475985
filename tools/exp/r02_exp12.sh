# K4 ceilings at the EP=8 per-GPU shape (16 x 4096) and EP=1 ragged rows: full kernel, no epilogue
# (debug 1), no operand loads (debug 32), neither (debug 33)
for d in 0 1 32 33; do
  MB_GEMM_DEBUG=$d timeout 120 python tools/bench_gemm.py --groups 16 --rows-per-group 4096 --only fwd1_swiglu,fwd2_store,dgrad_gated,dgrad_dx --iters 30 > gpurun_out/e12_g16_d$d.json 2>&1
  MB_GEMM_DEBUG=$d timeout 120 python tools/bench_gemm.py --zipf-rows --only fwd1_swiglu,dgrad_dx --iters 30 > gpurun_out/e12_zipf_d$d.json 2>&1
done
timeout 120 python tools/bench_gemm.py --groups 16 --rows-per-group 4096 --cublas --only none --iters 30 > gpurun_out/e12_cublas.json 2>&1
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm --format=csv
