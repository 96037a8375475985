O=fwd1_swiglu,fwd2_store,dgrad_gated,dgrad_dx,wgrad_w2,wgrad_w1
export MB_GEMM_PROF=1
python tools/bench_gemm.py --only $O --iters 1 --warmup 1 2>&1 | grep -v "^{" | tail -6
python tools/bench_gemm.py --only $O --iters 1 --warmup 1 --groups 16 --rows-per-group 4096 2>&1 | grep -v "^{" | tail -6
