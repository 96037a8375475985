# NVLink evidence for the row movers on a >= 2-GPU box (one process: GPU 0 -> GPU 1 rows).
python tools/nvlink_rows.py --blocks 28 > gpurun_out/nvl_rows_tma.json 2>&1; echo rows_tma=$?
python tools/nvlink_rows.py --blocks 0 > gpurun_out/nvl_rows_regs.json 2>&1; echo rows_regs=$?
ncu --query-metrics --chip gb100 2>/dev/null | grep -i "nvl" > gpurun_out/nvl_metric_names.txt
M=$(grep -oE "^nvl[a-z_]+__bytes" gpurun_out/nvl_metric_names.txt | sort -u | sed 's/$/.sum/' | paste -sd, -)
echo "metrics: $M"
ncu --metrics gpu__time_duration.sum,${M:-dram__bytes_read.sum} --clock-control none -k regex:"scatter|combine" \
    -c 8 --csv --log-file gpurun_out/r02_ncu_nvlink_rows.csv python tools/nvlink_rows.py --blocks 28 --iters 2 \
    > gpurun_out/ncu_nvl.log 2>&1; echo ncu=$?
