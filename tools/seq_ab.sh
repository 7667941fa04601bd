timeout 900 python -m pytest -x -q tests/test_gpu_parity.py tests/test_gpu_large.py tests/test_acceptance_gpu.py -k "tune" > gpurun_out/seq_t.log 2>&1; tail -3 gpurun_out/seq_t.log
bash tools/ab_env.sh c5 "" "BM_NW_SEQ=1" "BM_NW_SEQ=0" > gpurun_out/seq_ab.log 2>&1
cat gpurun_out/seq_ab.log
