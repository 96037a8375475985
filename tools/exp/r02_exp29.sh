# final code: EP=8 as 8 ranks on 4 GPUs (correctness only) + --check at the wide shapes (N=4)
bash tools/oversub8.sh
python -c "import json;d=json.loads(open('gpurun_out/o8_bench.json').read().strip().splitlines()[-1]);print('o8', d.get('n_gpus'), d['check']['ok'], d.get('oversubscribed'), d['config'])"
timeout 1200 python bench.py --gpus 4 --config qwen3-235b-a22b --group 2 --steps 3 --check --batches 1 --policies relibra \
    > gpurun_out/e29_235b.json 2> gpurun_out/e29_235b.err; echo b235=$?
timeout 1200 python bench.py --gpus 4 --config mixtral-8x7b --micro-batches 4 --steps 3 --check --batches 1 --policies relibra \
    > gpurun_out/e29_mixtral.json 2> gpurun_out/e29_mixtral.err; echo mixtral=$?
for f in e29_235b e29_mixtral; do python -c "
import json;d=json.loads(open('gpurun_out/$f.json').read().strip().splitlines()[-1])
print('$f', round(d['ms_per_step'],2), d['check']['ok'], {k:v.get('max_rel') for k,v in d['check'].items() if isinstance(v,dict)})"; done
