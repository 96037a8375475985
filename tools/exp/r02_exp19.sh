# pair (256-row tiles, half tiles for odd tails) vs single-CTA family (128-row tiles) on ragged / balanced rows
for v in pair single; do
  f=""; [ $v = single ] && f="--single"
  timeout 120 python tools/bench_gemm.py --zipf-rows --only fwd1_swiglu,fwd2_store,dgrad_gated,dgrad_dx --iters 30 $f > gpurun_out/e19_zipf_$v.json 2>&1
  timeout 120 python tools/bench_gemm.py --groups 16 --rows-per-group 4096 --only fwd1_swiglu,fwd2_store,dgrad_gated,dgrad_dx --iters 30 $f > gpurun_out/e19_g16_$v.json 2>&1
done
