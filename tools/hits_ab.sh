timeout 600 python -m pytest -x -q tests/test_gpu_parity.py -k "mixed or docs40 or 200x200 or tsv or host or skewed or sha256" > gpurun_out/hm_t.log 2>&1; tail -n 1 gpurun_out/hm_t.log
bash tools/ab_env.sh c3 "--c3-docs 200000" "BM_X=0" "BM_X=1" > gpurun_out/hm_ab.log 2>&1
bash tools/ab_env.sh c2 "" "BM_X=0" >> gpurun_out/hm_ab.log 2>&1
cat gpurun_out/hm_ab.log
