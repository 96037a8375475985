O=fwd1_swiglu,fwd2_store,dgrad_gated,dgrad_dx,wgrad_w2,wgrad_w1
for i in 1 2; do
python tools/bench_gemm.py --zipf-rows --only $O
python tools/bench_gemm.py --only $O
python tools/bench_gemm.py --only $O --groups 16 --rows-per-group 4096
done
