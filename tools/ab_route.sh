# routing A/B: fused tier vs banded tier for small documents
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/ab_smoke.log 2>&1
bash tools/ab_env.sh c3 "--c3-docs 200000" "BM_X=0" "BM_ROUTE=banded" "BM_FUSED_MAX_SMEM=20000" > gpurun_out/ab_route_c3.log 2>&1
bash tools/ab_env.sh c2 "" "BM_X=0" "BM_ROUTE=banded" > gpurun_out/ab_route_c2.log 2>&1
