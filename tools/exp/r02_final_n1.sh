# final N=1: default bench (as the driver runs it), --check run, reference arm
timeout 900 python bench.py > gpurun_out/f1_bench.json 2> gpurun_out/f1_bench.err; echo bench=$?
timeout 900 python bench.py --check --batches 1 > gpurun_out/f1_check.json 2> gpurun_out/f1_check.err; echo check=$?
timeout 900 python bench.py --impl reference > gpurun_out/f1_ref.json 2> gpurun_out/f1_ref.err; echo ref=$?
