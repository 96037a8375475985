# final-code ncu: launch list of one N=1 step (DRAM bytes per launch) + full captures of the two
# modes the pre-gated layout changed (dAct without the Act rewrite, fwd1 with the gate scale)
export MB_NVTX_STEP=1
ncu --nvtx --nvtx-include "mb_step/" --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
    --clock-control none --csv --log-file gpurun_out/r02_launches_step.csv \
    python bench.py --steps 1 --warmup 3 --repeats 1 --batches 1 --no-cpu-baseline --policies relibra \
    > gpurun_out/ncu_step.log 2>&1
echo launches_rc=$?
python tools/launch_summary.py gpurun_out/r02_launches_step.csv gpurun_out/r02_launches_step_summary.json \
    > gpurun_out/r02_launches_step_summary.txt 2>&1
cat gpurun_out/r02_launches_step_summary.txt | head -16
unset MB_NVTX_STEP
for m in dgrad_gated_noact fwd1_pregated; do
  f=""; [ $m = fwd1_pregated ] && f="--single"
  ncu --set full --clock-control none --import-source on -k regex:grouped_gemm -s 3 -c 1 \
      -o gpurun_out/r02_${m}_zipf -f python tools/bench_gemm.py --zipf-rows --only $m --iters 1 --warmup 3 $f \
      > gpurun_out/ncu_${m}.log 2>&1
  echo full_${m}_rc=$?
done
