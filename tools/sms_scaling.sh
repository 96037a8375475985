for sms in 148 112 74 38; do
  for d in 0 1; do
    echo "sms=$sms debug=$d $(MB_GEMM_SMS=$sms MB_GEMM_DEBUG=$d python tools/bench_gemm.py --only fwd1_swiglu,dgrad_dx --groups 16 --rows-per-group 4096)"
  done
done
