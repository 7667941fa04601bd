timeout 600 python -m pytest -x -q tests/test_gpu_parity.py -k "mixed_sizes" > gpurun_out/pers_t.log 2>&1; tail -1 gpurun_out/pers_t.log
bash tools/ab_env.sh c3 "--c3-docs 200000" "BM_X=0" "BM_SCORE_CTAS_PER_SM=3" "BM_SCORE_CTAS_PER_SM=3 BM_NW_WARPS_PER_SM=4" "BM_SCORE_CTAS_PER_SM=2 BM_NW_WARPS_PER_SM=4" "BM_SCORE_CTAS_PER_SM=3 BM_RING_CTAS_PER_SM=4 BM_NW_WARPS_PER_SM=4" "BM_SCORE_CTAS_PER_SM=3 BM_NW_WARPS_PER_SM=4 BM_DP_PRIO=1" > gpurun_out/pers_ab.log 2>&1
cat gpurun_out/pers_ab.log
