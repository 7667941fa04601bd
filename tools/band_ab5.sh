BM_BAND_FUSED=1 BM_BAND_MIN_ITEMS=1 timeout 600 python tests/par_walk_child.py 2026 > gpurun_out/b5_t.log 2>&1; tail -1 gpurun_out/b5_t.log
export BM_BAND_FUSED=1
bash tools/ab_wl.sh c3 "--c3-docs 200000" default bs0 bs1k bsarr0 bcpt4 > gpurun_out/band_ab5.log 2>&1
BM_BAND_FUSED=0 bash tools/ab_wl.sh c3 "--c3-docs 200000" default >> gpurun_out/band_ab5.log 2>&1
cat gpurun_out/band_ab5.log
