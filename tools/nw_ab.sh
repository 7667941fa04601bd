BM_LIB_PATH=tools/_prof/nwdirect.so timeout 600 python -m pytest -x -q tests/test_gpu_parity.py -k "mixed_sizes or tune" tests/test_gpu_large.py -k "tail or mixed or tune or c4" > gpurun_out/nw_t.log 2>&1; tail -2 gpurun_out/nw_t.log
bash tools/ab_wl.sh c3 "--c3-docs 200000" default nwdirect nwdirect16 nwdirect20 > gpurun_out/nw_ab.log 2>&1
bash tools/ab_wl.sh c5 "" default nwdirect >> gpurun_out/nw_ab.log 2>&1
bash tools/ab_wl.sh c4 "" default nwdirect >> gpurun_out/nw_ab.log 2>&1
cat gpurun_out/nw_ab.log
