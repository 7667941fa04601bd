export BM_LIB_PATH=tools/_prof/cpt2.so
bash tools/ab_env.sh c3 "--c3-docs 200000" "BM_NW_STAGGER=512" "BM_NW_STAGGER=2048" "BM_NW_STAGGER=16384" > gpurun_out/band_ab4.log 2>&1
export BM_LIB_PATH=tools/_prof/cpt2s8.so
bash tools/ab_env.sh c3 "--c3-docs 200000" "BM_NW_STAGGER=512" >> gpurun_out/band_ab4.log 2>&1
cat gpurun_out/band_ab4.log
