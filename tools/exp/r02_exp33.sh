# replica wgrad with K split in halves (MB_REPLICA_SPLIT_K=1): parity (multi-rank tests) + N=4 / N=2 A/B
MB_REPLICA_SPLIT_K=1 timeout 900 python -m pytest tests/test_multirank_gpu.py -q -x -p no:cacheprovider > gpurun_out/e33_tests.log 2>&1; echo tests=$?; tail -1 gpurun_out/e33_tests.log
bash tools/ab_env.sh 4 "MB_REPLICA_SPLIT_K=1" "MB_REPLICA_SPLIT_K=0" 3
bash tools/ab_env.sh 2 "MB_REPLICA_SPLIT_K=1" "MB_REPLICA_SPLIT_K=0" 2
