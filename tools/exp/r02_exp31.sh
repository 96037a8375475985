# replica weight gradients on every SM (MB_REPLICA_WGRAD_ALL_SMS=1) vs the GEMM's share: N=4, N=2
bash tools/ab_env.sh 4 "MB_REPLICA_WGRAD_ALL_SMS=1" "MB_REPLICA_WGRAD_ALL_SMS=0" 3
bash tools/ab_env.sh 2 "MB_REPLICA_WGRAD_ALL_SMS=1" "MB_REPLICA_WGRAD_ALL_SMS=0" 2
