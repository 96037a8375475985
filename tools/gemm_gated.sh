timeout 300 python -m pytest tests/test_gemm_gpu.py tests/test_layer_gpu.py -x -q 2>&1 | tail -2
for i in 1 2; do
python tools/bench_gemm.py --only dgrad_gated,dgrad_dswiglu --groups 16 --rows-per-group 4096
python tools/bench_gemm.py --only dgrad_gated,dgrad_dswiglu
python tools/bench_gemm.py --only dgrad_gated --zipf-rows
done
