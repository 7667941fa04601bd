timeout 240 python -m pytest -x -q tests/test_gpu_large.py -k "c4_full" > gpurun_out/ovl_t.log 2>&1; echo "rc=$?"; tail -2 gpurun_out/ovl_t.log
timeout 600 python -m pytest -x -q tests/test_gpu_large.py tests/test_gpu_parity.py -k "c4 or long_pair or mixed or tail or band_parallel" > gpurun_out/ovl_t2.log 2>&1; echo "rc=$?"; tail -2 gpurun_out/ovl_t2.log
timeout 300 bash tools/ab_env.sh c4 "" "BM_DP_OVERLAP=1" "BM_DP_OVERLAP=0" > gpurun_out/ovl_ab.log 2>&1
cat gpurun_out/ovl_ab.log
