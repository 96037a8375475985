# final code on one 4-GPU box: GPU suite + smoke, N=1 / 2 / 4 bench lines, N=4 --check, N=1 ncu launch list
timeout 1500 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/g4_pytest.log 2>&1; echo pytest=$?
tail -2 gpurun_out/g4_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/g4_smoke.log 2>&1; echo smoke=$?
CUDA_VISIBLE_DEVICES=0 timeout 900 python bench.py > gpurun_out/g4_n1.json 2> gpurun_out/g4_n1.err; echo n1=$?
timeout 900 python bench.py --gpus 2 > gpurun_out/g4_n2.json 2> gpurun_out/g4_n2.err; echo n2=$?
timeout 1200 python bench.py --gpus 4 > gpurun_out/g4_n4.json 2> gpurun_out/g4_n4.err; echo n4=$?
timeout 900 python bench.py --gpus 4 --check --batches 1 --policies relibra > gpurun_out/g4_n4_check.json 2> gpurun_out/g4_n4_check.err; echo n4check=$?
CUDA_VISIBLE_DEVICES=0 timeout 600 python bench.py --impl reference > gpurun_out/g4_ref.json 2> gpurun_out/g4_ref.err; echo ref=$?
for f in g4_n1 g4_n2 g4_n4 g4_n4_check; do python -c "
import json;d=json.loads(open('gpurun_out/$f.json').read().strip().splitlines()[-1]);b=d.get('balance',{})
print('$f', round(d['ms_per_step'],3), round(d['value']/1e6,3), d['roofline']['frac'], d['clocks']['sm_mhz'], b.get('speedup_vs_static'), b.get('frac_of_balanced'), (d.get('check') or {}).get('ok'))"; done
export MB_NVTX_STEP=1
CUDA_VISIBLE_DEVICES=0 ncu --nvtx --nvtx-include "mb_step/" --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
    --clock-control none --csv --log-file gpurun_out/r02_launches_step.csv \
    python bench.py --steps 1 --warmup 3 --repeats 1 --batches 1 --no-cpu-baseline --policies relibra \
    > gpurun_out/ncu_step.log 2>&1
echo launches_rc=$?
python tools/launch_summary.py gpurun_out/r02_launches_step.csv gpurun_out/r02_launches_step_summary.json \
    > gpurun_out/r02_launches_step_summary.txt 2>&1
head -8 gpurun_out/r02_launches_step_summary.txt
