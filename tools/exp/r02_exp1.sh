set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv
python tools/bench_gemm.py --zipf-rows --iters 20 > gpurun_out/e1_zipf148.json 2>&1
MB_GEMM_SMS=128 python tools/bench_gemm.py --zipf-rows --iters 20 > gpurun_out/e1_zipf128.json 2>&1
python tools/bench_gemm.py --groups 128 --rows-per-group 512 --cublas --iters 20 > gpurun_out/e1_bal148.json 2>&1
python tools/bench_gemm.py --groups 16 --rows-per-group 4096 --iters 20 > gpurun_out/e1_g16.json 2>&1
python tools/bench_gemm.py --groups 128 --rows-per-group 512 --only dgrad_gated --iters 20 > gpurun_out/e1_gated.json 2>&1
for m in fwd1_swiglu fwd2_store dgrad_gated dgrad_dx wgrad_w1; do
MB_KERNELS_LIB=libmb_sm100_prof.so MB_GEMM_PROF=1 python tools/bench_gemm.py --zipf-rows --only $m --iters 2 --warmup 1 > gpurun_out/e1_prof_$m.log 2>&1
done
timeout 600 python bench.py --steps 10 --warmup 3 --policies relibra,static > gpurun_out/e1_bench.json 2> gpurun_out/e1_bench.err
