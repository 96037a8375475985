for sms in 120 112 104; do
MB_GEMM_SMS=$sms python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 2971$((sms%10)) bench.py --gpus 4 --steps 6 --policies relibra > gpurun_out/n4s_$sms.json 2> gpurun_out/n4s_$sms.err; echo rc=$?
MB_GEMM_SMS=$sms python bench.py --steps 6 --policies relibra --no-cpu-baseline > gpurun_out/n1s_$sms.json 2> gpurun_out/n1s_$sms.err; echo rc=$?
done
