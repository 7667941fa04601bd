timeout 900 python -m pytest -x -q tests/test_gpu_large.py tests/test_gpu_parity.py -k "large or mixed or tune or c4" > gpurun_out/ver_t.log 2>&1; tail -1 gpurun_out/ver_t.log
bash tools/ab_wl.sh c3 "--c3-docs 200000" default base_r02 default base_r02 > gpurun_out/ver_ab.log 2>&1
cat gpurun_out/ver_ab.log
