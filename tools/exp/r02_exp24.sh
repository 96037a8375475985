# GEMMs on an own high-priority stream (MB_COMPUTE_PRIORITY=high) vs the caller's stream: N=1, N=4
MB_COMPUTE_PRIORITY=high timeout 600 python -m pytest tests/test_layer_gpu.py -q -x -p no:cacheprovider > gpurun_out/e24_layer.log 2>&1; echo layer=$?
CUDA_VISIBLE_DEVICES=0 bash -c 'for v in hi lo hi lo; do
  e=X=1; [ $v = hi ] && e=MB_COMPUTE_PRIORITY=high
  env $e timeout 300 python bench.py --policies relibra --batches 1 --repeats 3 --no-cpu-baseline > gpurun_out/e24_n1_$v.json 2>> gpurun_out/e24_bench.err
  python -c "import json;d=json.loads(open(\"gpurun_out/e24_n1_$v.json\").read().strip().splitlines()[-1]);print(\"n1 $v\", round(d[\"ms_per_step\"],3), d[\"roofline\"][\"frac\"])"
done'
for v in hi lo; do
  e=X=1; [ $v = hi ] && e=MB_COMPUTE_PRIORITY=high
  env $e timeout 900 python bench.py --gpus 4 --policies relibra --batches 1 --repeats 3 > gpurun_out/e24_n4_$v.json 2>> gpurun_out/e24_bench.err
  python -c "import json;d=json.loads(open('gpurun_out/e24_n4_$v.json').read().strip().splitlines()[-1]);print('n4 $v', round(d['ms_per_step'],3), d['roofline']['frac'])"
done
