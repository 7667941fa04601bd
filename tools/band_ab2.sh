bash tools/ab_wl.sh c3 "--c3-docs 200000" default noalloc0 minb6 slots2 > gpurun_out/band_ab2.log 2>&1
bash tools/ab_env.sh c3 "--c3-docs 200000" "BM_BAND_FUSED=0" >> gpurun_out/band_ab2.log 2>&1
BM_LIB_PATH=tools/_prof/noalloc0.so bash tools/ab_env.sh c3 "--c3-docs 200000" "BM_BAND_FUSED=0" >> gpurun_out/band_ab2.log 2>&1
cat gpurun_out/band_ab2.log
