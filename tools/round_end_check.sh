timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pt_final.log 2>&1; echo pytest=$?
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_final.log 2>&1; echo smoke=$?
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
timeout 300 $TR --master-port 29951 tools/mgpu_check.py --config qwen3-30b-a3b --tokens 2048 --micro-batches 3 --group 2 --steps 2 > gpurun_out/c4_final.log 2>&1; echo chk=$?
timeout 300 $TR --master-port 29953 tools/mgpu_migrate.py --config qwen3-30b-a3b --tokens 1024 > gpurun_out/m4_final.log 2>&1; echo mig=$?
bash tools/final_evidence.sh > gpurun_out/fin.log 2>&1; echo fin=$?
