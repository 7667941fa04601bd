timeout 600 python -m pytest -x -q tests/test_gpu_parity.py -k "mixed or 200x200 or stress or docs40" > gpurun_out/occ_t.log 2>&1; tail -n 1 gpurun_out/occ_t.log
bash tools/ab_wl.sh c3 "--c3-docs 200000" default hd9 hd12 hk10 hk14 rg7 rg8 > gpurun_out/occ_ab.log 2>&1
bash tools/ab_wl.sh c2 "" default rg7 rg8 hk10 hk14 >> gpurun_out/occ_ab.log 2>&1
cat gpurun_out/occ_ab.log
