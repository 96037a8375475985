# shared layer-shared replica buffer across layers: multi-rank + layer suites, smoke
timeout 1200 python -m pytest tests/test_multirank_gpu.py tests/test_layer_gpu.py -q -p no:cacheprovider > gpurun_out/e16_pytest.log 2>&1; echo pytest=$?
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/e16_smoke.log 2>&1; echo smoke=$?
