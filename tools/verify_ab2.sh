timeout 600 python -m pytest -x -q tests/test_gpu_parity.py -k "mixed or docs40 or 200x200 or tsv or host" > gpurun_out/ver2_t.log 2>&1; tail -1 gpurun_out/ver2_t.log
bash tools/ab_wl.sh c3 "--c3-docs 200000" default base_r02 ring_cpt2 nalloc0b default base_r02 > gpurun_out/ver2_ab.log 2>&1
bash tools/ab_wl.sh c2 "" default base_r02 ring_cpt2 >> gpurun_out/ver2_ab.log 2>&1
cat gpurun_out/ver2_ab.log
