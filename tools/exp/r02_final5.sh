# final code on a 1-GPU box: full GPU suite + smoke + the default bench line + reference arm
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/g5_pytest.log 2>&1; echo pytest=$?
tail -2 gpurun_out/g5_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/g5_smoke.log 2>&1; echo smoke=$?
timeout 900 python bench.py > gpurun_out/g5_n1.json 2> gpurun_out/g5_n1.err; echo n1=$?
python -c "
import json;d=json.loads(open('gpurun_out/g5_n1.json').read().strip().splitlines()[-1]);b=d['balance']
print('n1', round(d['ms_per_step'],3), round(d['value']/1e6,3), d['roofline']['frac'], d['clocks'], d['e2e']['value'], b['relibra']['ms_per_step'], b['static']['ms_per_step'], b['eplb_like']['ms_per_step'])"
