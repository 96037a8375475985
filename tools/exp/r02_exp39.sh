# last combine ahead of the third-to-last un-permute (MB_EARLY_LAST_COMBINE=1) + ring guard
timeout 1200 python -m pytest tests/test_multirank_gpu.py -q -x -p no:cacheprovider > gpurun_out/e39_tests.log 2>&1; echo tests=$?; tail -1 gpurun_out/e39_tests.log
timeout 900 python bench.py --gpus 4 --check --batches 1 --policies relibra > gpurun_out/e39_check.json 2> gpurun_out/e39_check.err; echo check=$?
python -c "import json;d=json.loads(open('gpurun_out/e39_check.json').read().strip().splitlines()[-1]);print('check', d['ms_per_step'], d['check']['ok'])"
bash tools/ab_env.sh 4 "MB_EARLY_LAST_COMBINE=1" "MB_EARLY_LAST_COMBINE=0" 3
bash tools/ab_env.sh 2 "MB_EARLY_LAST_COMBINE=1" "MB_EARLY_LAST_COMBINE=0" 2
