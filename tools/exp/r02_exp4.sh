# 4-GPU box: real multi-GPU parity + bench N=4 (replica sets 2 / 1, micro_batch wgrad) + N=2
nvidia-smi -L
timeout 900 python -m pytest tests/test_multirank_gpu.py -q -p no:cacheprovider -k real > gpurun_out/e4_pytest.log 2>&1; echo pytest=$?
timeout 900 python bench.py --gpus 4 > gpurun_out/e4_n4.json 2> gpurun_out/e4_n4.err; echo n4=$?
MB_REPLICA_SETS=1 timeout 900 python bench.py --gpus 4 --policies relibra --batches 1 > gpurun_out/e4_n4_sets1.json 2> gpurun_out/e4_n4_sets1.err; echo n4s1=$?
timeout 900 python bench.py --gpus 4 --policies relibra --batches 1 --wgrad-mode micro_batch > gpurun_out/e4_n4_mbw.json 2> gpurun_out/e4_n4_mbw.err; echo n4mb=$?
timeout 900 python bench.py --gpus 2 --batches 1 > gpurun_out/e4_n2.json 2> gpurun_out/e4_n2.err; echo n2=$?
