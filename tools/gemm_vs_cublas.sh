O=fwd1_swiglu,fwd2_store,dgrad_gated,dgrad_dx,wgrad_w2,wgrad_w1
python tools/bench_gemm.py --only $O --groups 16 --rows-per-group 4096 --cublas
python tools/bench_gemm.py --only $O --cublas
python tools/bench_gemm.py --only $O --groups 16 --rows-per-group 4096 --cublas
