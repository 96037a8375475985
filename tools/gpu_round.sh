# one-GPU evidence pass: parity tests, smoke, bench line, ncu launch list + data-plane kernel metrics
mkdir -p gpurun_out
python -m pytest tests -m gpu -x -q > gpurun_out/pt_gpu.log 2>&1; echo pytest_rc=$? | tee -a gpurun_out/pt_gpu.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke_rc=$?
python bench.py > gpurun_out/bench_n1.json 2> gpurun_out/bench_n1.err; echo bench_rc=$?
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_n1.csv \
    python bench.py --steps 1 --warmup 1 --no-cpu-baseline --policies relibra > gpurun_out/ncu_launch.log 2>&1; echo ncu1_rc=$?
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__throughput.avg.pct_of_peak_sustained_elapsed \
    --clock-control none -k regex:"histogram|permute|scatter|combine|zero_pad|chunk_scan" -c 40 --csv \
    --log-file gpurun_out/dataplane_n1.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline --policies relibra \
    > gpurun_out/ncu_dp.log 2>&1; echo ncu2_rc=$?
