# 4-GPU box: full GPU suite (device dispatch tables, real multi-GPU replica step)
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider --durations=10 > gpurun_out/e8_pytest.log 2>&1; echo pytest=$?
