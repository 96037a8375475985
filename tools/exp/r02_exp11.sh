# 4-GPU box: bench N=4 and N=2 with dynamic tile scheduling + two-problem wgrad
timeout 1200 python bench.py --gpus 4 > gpurun_out/e11_n4.json 2> gpurun_out/e11_n4.err; echo n4=$?
timeout 900 python bench.py --gpus 2 > gpurun_out/e11_n2.json 2> gpurun_out/e11_n2.err; echo n2=$?
MB_COMM_SMS=20 timeout 900 python bench.py --gpus 4 --policies relibra --batches 1 > gpurun_out/e11_n4_c20.json 2> gpurun_out/e11_n4_c20.err; echo n4c20=$?
MB_COMM_SMS=36 timeout 900 python bench.py --gpus 4 --policies relibra --batches 1 > gpurun_out/e11_n4_c36.json 2> gpurun_out/e11_n4_c36.err; echo n4c36=$?
