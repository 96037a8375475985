for d in 0 64 32; do
  echo "debug=$d $(MB_GEMM_DEBUG=$d python tools/bench_gemm.py --only dgrad_dx --groups 16 --rows-per-group 4096 2>&1 | tail -1)"
done
