# ncu --set full of the TMA row movers and the register movers (one GPU, bench_rows parity pass)
ncu --set full --clock-control none --import-source on -k regex:"scatter_rows|combine_rows" -c 9 \
    -o gpurun_out/r01_rows_full2 -f python tools/bench_rows.py --blocks 32 --iters 1 > gpurun_out/ncu_rows.log 2>&1
echo rc=$?
ncu -i gpurun_out/r01_rows_full2.ncu-rep --page raw --csv \
    --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,launch__grid_size,launch__block_size,sm__throughput.avg.pct_of_peak_sustained_elapsed,dram__throughput.avg.pct_of_peak_sustained_elapsed \
    > gpurun_out/r01_rows_raw2.csv 2>&1
echo rc2=$?
