bash tools/ab_env.sh c2 "" "BM_X=0" "BM_CHUNK_CELLS=8388608 BM_FIRST_CHUNK_CELLS=1048576" "BM_CHUNK_CELLS=8388608 BM_FIRST_CHUNK_CELLS=2097152" "BM_CHUNK_CELLS=12582912 BM_FIRST_CHUNK_CELLS=1048576" > gpurun_out/chunk_ab2.log 2>&1
bash tools/ab_env.sh c3 "--c3-docs 200000" "BM_X=0" "BM_FIRST_CHUNK_CELLS=1048576" >> gpurun_out/chunk_ab2.log 2>&1
bash tools/ab_env.sh c4 "" "BM_X=0" "BM_FIRST_CHUNK_CELLS=1048576" >> gpurun_out/chunk_ab2.log 2>&1
cat gpurun_out/chunk_ab2.log
