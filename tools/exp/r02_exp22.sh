# 4-GPU box: full GPU suite + smoke on the current kernels
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/e22_pytest.log 2>&1; echo pytest=$?
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/e22_smoke.log 2>&1; echo smoke=$?
