BM_LIB_PATH=tools/_prof/cpt2.so timeout 600 python -m pytest -x -q tests/test_gpu_parity.py -k "mixed_sizes or skewed" tests/test_gpu_large.py -k "tail or mixed or skewed" > gpurun_out/band_t3.log 2>&1; tail -2 gpurun_out/band_t3.log
bash tools/ab_wl.sh c3 "--c3-docs 200000" default cpt2 cpt2m4 > gpurun_out/band_ab3.log 2>&1
cat gpurun_out/band_ab3.log
