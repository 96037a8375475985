# Mixtral-8x7B at N=4: two replica sets (new default for 336 MiB experts) vs one
timeout 1500 python bench.py --gpus 4 --config mixtral-8x7b --repeats 2 --batches 1 > gpurun_out/e18_mixtral_sets2.json 2> gpurun_out/e18_m2.err; echo sets2=$?
MB_REPLICA_SETS=1 timeout 1200 python bench.py --gpus 4 --config mixtral-8x7b --repeats 2 --batches 1 --policies relibra > gpurun_out/e18_mixtral_sets1.json 2> gpurun_out/e18_m1.err; echo sets1=$?
