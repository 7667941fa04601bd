timeout 600 python -m pytest -x -q tests/test_gpu_parity.py -k "mixed_sizes or skewed or docs40 or 200x200 or stress or host_entry" > gpurun_out/ring_t.log 2>&1; tail -2 gpurun_out/ring_t.log
BM_LIB_PATH=tools/_prof/ring_cpt1.so timeout 600 python -m pytest -x -q tests/test_gpu_parity.py -k "mixed_sizes" > gpurun_out/ring_t1.log 2>&1; tail -2 gpurun_out/ring_t1.log
bash tools/ab_wl.sh c2 "" default ring_cpt1 ring_old > gpurun_out/ring_ab.log 2>&1
bash tools/ab_wl.sh c3 "--c3-docs 200000" default ring_cpt1 ring_old >> gpurun_out/ring_ab.log 2>&1
cat gpurun_out/ring_ab.log
