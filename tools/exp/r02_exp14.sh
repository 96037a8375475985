# 4-GPU box: GPU suite + smoke after the kernel changes, and step timelines at N=4 / N=1
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/e14_pytest.log 2>&1; echo pytest=$?
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/e14_smoke.log 2>&1; echo smoke=$?
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 600 $TR --nproc-per-node 4 --master-port 29961 tools/step_timeline.py > gpurun_out/e14_timeline_n4.jsonl 2> gpurun_out/e14_timeline_n4.err; echo tl4=$?
timeout 600 python tools/step_timeline.py > gpurun_out/e14_timeline_n1.jsonl 2> gpurun_out/e14_timeline_n1.err; echo tl1=$?
