timeout 600 python -m pytest -x -q tests/test_gpu_parity.py -k "mixed_sizes or docs40 or tsv" > gpurun_out/r2_t.log 2>&1; tail -1 gpurun_out/r2_t.log
bash tools/ab_wl.sh c2 "" default rs0 rs128 rs512 > gpurun_out/ring_ab2.log 2>&1
bash tools/ab_wl.sh c3 "--c3-docs 200000" default rs0 rs128 >> gpurun_out/ring_ab2.log 2>&1
cat gpurun_out/ring_ab2.log
