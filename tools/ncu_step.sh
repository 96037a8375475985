# launch list of our kernels over the bench step (one GPU) + DRAM bytes per launch
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    -k regex:"grouped_gemm|histogram|permute|scatter|combine|zero_pad|chunk_scan|accumulate|peer_barrier" \
    -c 1500 --csv --log-file gpurun_out/r01_launches_step2.csv \
    python bench.py --steps 1 --warmup 1 --no-cpu-baseline --policies relibra > gpurun_out/ncu_step.log 2>&1
echo rc=$?
