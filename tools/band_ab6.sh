export BM_BAND_FUSED=1
BM_LIB_PATH=tools/_prof/bp1.so BM_BAND_MIN_ITEMS=1 timeout 300 python tests/par_walk_child.py 2026 > gpurun_out/b6_t1.log 2>&1; tail -1 gpurun_out/b6_t1.log
BM_LIB_PATH=tools/_prof/bp1k2.so BM_BAND_MIN_ITEMS=1 timeout 300 python tests/par_walk_child.py 7 > gpurun_out/b6_t2.log 2>&1; tail -1 gpurun_out/b6_t2.log
BM_BAND_MIN_ITEMS=1 BM_PAR_WALK_MIN=600 timeout 300 python tests/par_walk_child.py 2026 > gpurun_out/b6_t3.log 2>&1; tail -1 gpurun_out/b6_t3.log
timeout 900 bash tools/ab_wl.sh c3 "--c3-docs 200000" default bp1 bp1k2 bp2 bp2k2 bp4 > gpurun_out/band_ab6.log 2>&1
BM_BAND_FUSED=0 timeout 300 bash tools/ab_wl.sh c3 "--c3-docs 200000" default >> gpurun_out/band_ab6.log 2>&1
cat gpurun_out/band_ab6.log
