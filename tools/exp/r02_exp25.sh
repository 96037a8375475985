# pre-gated activation (gate*act from the gate/up GEMM, plain-sum combine, no Act rewrite in dAct)
timeout 900 python -m pytest tests/test_gemm_gpu.py tests/test_layer_gpu.py -q -x -p no:cacheprovider > gpurun_out/e25_tests.log 2>&1; echo tests=$?
tail -3 gpurun_out/e25_tests.log
for i in 1 2; do
timeout 300 python tools/bench_gemm.py --zipf-rows --only dgrad_gated,dgrad_gated_noact 2>&1 | tail -1
timeout 300 python tools/bench_gemm.py --zipf-rows --single --only fwd1_swiglu,fwd1_pregated 2>&1 | tail -1
done
bash tools/ab_env.sh 1 "MB_PREGATE=1" "MB_PREGATE=0" 3
timeout 600 python bench.py --check --batches 1 --policies relibra --no-cpu-baseline > gpurun_out/e25_check.json 2> gpurun_out/e25_check.err
python -c "import json;d=json.loads(open('gpurun_out/e25_check.json').read().strip().splitlines()[-1]);print('check', d['ms_per_step'], d['check']['ok'], {k:v.get('max_rel') for k,v in d['check'].items() if isinstance(v,dict)})"
