export MB_GEMM_PROF=1
for m in fwd1_swiglu dgrad_gated dgrad_dx fwd2_store; do
python tools/bench_gemm.py --only $m --iters 1 --warmup 1 --groups 16 --rows-per-group 4096 2>&1 | grep gemm-prof | tail -1
python tools/bench_gemm.py --only $m --iters 1 --warmup 1 2>&1 | grep gemm-prof | tail -1
done
