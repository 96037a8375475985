# GPU suite + smoke + default bench (with --check) after the replica-path redesign
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider --durations=20 > gpurun_out/e3_pytest.log 2>&1; echo pytest=$?
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/e3_smoke.log 2>&1; echo smoke=$?
timeout 900 python bench.py --check > gpurun_out/e3_bench.json 2> gpurun_out/e3_bench.err; echo bench=$?
