# bm_mine group size (BM_GROUP_CELLS): smaller groups rotate over the three streams, so one
# group's latency-bound join (hits_kernel) overlaps another's issue-bound ring kernel
bash tools/ab_env.sh c2 "" "BM_GROUP_CELLS=1073741824" "BM_GROUP_CELLS=33554432" "BM_GROUP_CELLS=16777216" "BM_GROUP_CELLS=8388608" > gpurun_out/group_ab.log 2>&1
bash tools/ab_env.sh c3 "--c3-docs 200000" "BM_GROUP_CELLS=1073741824" "BM_GROUP_CELLS=268435456" "BM_GROUP_CELLS=134217728" >> gpurun_out/group_ab.log 2>&1
bash tools/ab_env.sh c5 "" "BM_GROUP_CELLS=1073741824" "BM_GROUP_CELLS=33554432" >> gpurun_out/group_ab.log 2>&1
cat gpurun_out/group_ab.log
