# last code state: EP=8 as 8 ranks on 4 GPUs (correctness of the reordered tail at EP=8)
bash tools/oversub8.sh
python -c "import json;d=json.loads(open('gpurun_out/o8_bench.json').read().strip().splitlines()[-1]);print('o8', d.get('n_gpus'), d['check']['ok'], d['config']['ep'])"
