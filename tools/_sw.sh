bash tools/ab_env.sh 4 "MB_X=1" "MB_GEMM_SMS=124 MB_COMM_BLOCKS=24" 1 > gpurun_out/sw4.log 2>&1
bash tools/ab_env.sh 4 "MB_GEMM_SMS=128 MB_COMM_BLOCKS=20" "MB_COMBINE_ENGINE=tma" 1 >> gpurun_out/sw4.log 2>&1
bash tools/ab_env.sh 1 "MB_X=1" "MB_ROW_MOVERS=tma MB_GEMM_SMS=136 MB_COMM_BLOCKS=12" 1 > gpurun_out/sw1.log 2>&1
bash tools/ab_env.sh 1 "MB_ROW_MOVERS=tma MB_GEMM_SMS=132 MB_COMM_BLOCKS=16" "MB_ROW_MOVERS=tma MB_GEMM_SMS=140 MB_COMM_BLOCKS=8" 1 >> gpurun_out/sw1.log 2>&1
