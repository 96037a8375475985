TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
timeout 300 $TR --master-port 29921 bench.py --gpus 4 --trace tests/golden/io/small/trace --plans tests/golden/io/small/plans --policies relibra,static,balanced_oracle --steps 3 > gpurun_out/tr_plans.json 2> gpurun_out/tr_plans.err; echo plans=$?
timeout 300 $TR --master-port 29922 bench.py --gpus 4 --trace tests/golden/io/small/trace --policies relibra,static --steps 3 > gpurun_out/tr_plan.json 2> gpurun_out/tr_plan.err; echo planned=$?
timeout 300 $TR --master-port 29923 tools/mgpu_migrate.py --config qwen3-30b-a3b --tokens 1024 > gpurun_out/mig_q2.log 2>&1; echo mig=$?
