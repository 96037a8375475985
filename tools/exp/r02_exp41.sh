# reordered schedule tail at N=1 (no replicas): interleaved A/B
bash tools/ab_env.sh 1 "MB_EARLY_LAST_COMBINE=1" "MB_EARLY_LAST_COMBINE=0" 4
