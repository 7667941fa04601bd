BM_LIB_PATH=tools/_prof/ex16.so timeout 600 python -m pytest -x -q tests/test_gpu_large.py tests/test_gpu_parity.py -k "tail or band_parallel or mixed or c4 or extract" > gpurun_out/ex_t.log 2>&1; tail -n 1 gpurun_out/ex_t.log
bash tools/ab_wl.sh c3 "--c3-docs 200000" default ex16 default ex16 > gpurun_out/ex_ab.log 2>&1
bash tools/ab_wl.sh c4 "" default ex16 >> gpurun_out/ex_ab.log 2>&1
cat gpurun_out/ex_ab.log
