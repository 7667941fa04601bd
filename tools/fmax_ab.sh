bash tools/ab_env.sh c3 "--c3-docs 200000" "BM_FUSED_MAX_SMEM=65536" "BM_FUSED_MAX_SMEM=98304" "BM_FUSED_MAX_SMEM=131072" "BM_FUSED_MAX_SMEM=49152" > gpurun_out/fmax_ab.log 2>&1
cat gpurun_out/fmax_ab.log
