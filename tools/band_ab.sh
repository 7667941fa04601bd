timeout 600 python -m pytest -x -q tests/test_gpu_parity.py -k "mixed_sizes or long_sentences or skewed or host_entry" tests/test_gpu_large.py > gpurun_out/band_tests.log 2>&1; tail -2 gpurun_out/band_tests.log
bash tools/ab_env.sh c3 "--c3-docs 200000" "BM_BAND_FUSED=1" "BM_BAND_FUSED=0" > gpurun_out/band_ab_c3.log 2>&1
bash tools/ab_env.sh c4 "" "BM_BAND_FUSED=1" > gpurun_out/band_ab_c4.log 2>&1
cat gpurun_out/band_ab_c3.log gpurun_out/band_ab_c4.log
