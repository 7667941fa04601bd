bash tools/ab_env.sh c3 "--c3-docs 200000" "BM_DP_PRIO=0" "BM_DP_PRIO=1" "BM_DP_PRIO=1 BM_NW_WARPS_PER_SM=4" "BM_DP_PRIO=1 BM_NW_WARPS_PER_SM=6" "BM_DP_PRIO=0 BM_NW_WARPS_PER_SM=6" > gpurun_out/prio_ab.log 2>&1
cat gpurun_out/prio_ab.log
