# final code on one 4-GPU box: full GPU suite + smoke, then N=1 / N=2 / N=4 bench lines, N=4 --check
timeout 1500 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/g3_pytest.log 2>&1; echo pytest=$?
tail -2 gpurun_out/g3_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/g3_smoke.log 2>&1; echo smoke=$?
CUDA_VISIBLE_DEVICES=0 timeout 900 python bench.py > gpurun_out/g3_n1.json 2> gpurun_out/g3_n1.err; echo n1=$?
timeout 900 python bench.py --gpus 2 > gpurun_out/g3_n2.json 2> gpurun_out/g3_n2.err; echo n2=$?
timeout 1200 python bench.py --gpus 4 > gpurun_out/g3_n4.json 2> gpurun_out/g3_n4.err; echo n4=$?
timeout 900 python bench.py --gpus 4 --check --batches 1 --policies relibra > gpurun_out/g3_n4_check.json 2> gpurun_out/g3_n4_check.err; echo n4check=$?
for f in g3_n1 g3_n2 g3_n4 g3_n4_check; do python -c "
import json;d=json.loads(open('gpurun_out/$f.json').read().strip().splitlines()[-1]);b=d.get('balance',{})
print('$f', round(d['ms_per_step'],3), round(d['value']/1e6,3), d['roofline']['frac'], d['clocks']['sm_mhz'], b.get('speedup_vs_static'), b.get('frac_of_balanced'), (d.get('check') or {}).get('ok'))"; done
