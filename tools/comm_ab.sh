run1() { env "$@" python bench.py --steps 6 --policies relibra --no-cpu-baseline > gpurun_out/cab_n1_$TAG.json 2>/dev/null; }
run4() { env "$@" python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port $((29800+RANDOM%100)) bench.py --gpus 4 --steps 6 --policies relibra > gpurun_out/cab_n4_$TAG.json 2>/dev/null; }
TAG=A; run1 X=1; run4 X=1
TAG=B; run1 MB_COMM_SMEM=32768; run4 MB_COMM_SMEM=32768
TAG=C; run1 MB_COMM_SMEM=32768 MB_GEMM_SMS=136; run4 MB_COMM_SMEM=32768 MB_GEMM_SMS=132
TAG=D; run1 MB_COMM_SMEM=32768 MB_GEMM_SMS=140; run4 MB_COMM_SMEM=32768 MB_GEMM_SMS=128
TAG=E; run1 MB_GEMM_SMS=148; run4 MB_COMM_SMEM=32768 MB_GEMM_SMS=136
echo done
