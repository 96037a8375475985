# wgrad operand loads with an L2 evict_last hint (libmb_sm100_wlast.so) vs default: DRAM bytes of
# the step's wgrad launch (ncu launch list) and the step time (interleaved A/B)
export MB_NVTX_STEP=1
for L in libmb_sm100.so libmb_sm100_wlast.so; do
MB_KERNELS_LIB=$L ncu --nvtx --nvtx-include "mb_step/" -k regex:grouped_gemm_pair --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
    --clock-control none --csv --log-file gpurun_out/e28_$L.csv \
    python bench.py --steps 1 --warmup 3 --repeats 1 --batches 1 --no-cpu-baseline --policies relibra > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/e28_$L.csv gpurun_out/e28_$L.json 2>&1 | head -4
done
unset MB_NVTX_STEP
bash tools/ab_env.sh 1 "MB_KERNELS_LIB=libmb_sm100.so" "MB_KERNELS_LIB=libmb_sm100_wlast.so" 3
# dAct epilogue decomposition (profiling flags): full, no H loads, no dH stores, neither, no epilogue
for d in 0 128 256 384 1; do
echo "debug=$d"; MB_GEMM_DEBUG=$d timeout 300 python tools/bench_gemm.py --zipf-rows --only dgrad_gated_noact 2>&1 | tail -1
done
