for d in 0 1 2 4; do
echo "debug=$d"
MB_GEMM_DEBUG=$d python tools/bench_gemm.py --only fwd1_swiglu,fwd2_store,dgrad_dx,dgrad_gated --groups 16 --rows-per-group 4096
done
