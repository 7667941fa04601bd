CMD="python bench.py --workload c3 --c3-docs 20000 --steps 1 --warmup 1 --extras none --no-cpu"
$CMD > gpurun_out/band_p.log 2>&1 || exit 1
ncu --set full --import-source on --clock-control none -k regex:"mine_band|score_hits|nw_band" -c 3 -o gpurun_out/band_full $CMD > gpurun_out/band_ncu.log 2>&1
BM_BAND_FUSED=0 ncu --set full --import-source on --clock-control none -k regex:"score_hits|nw_band" -c 2 -o gpurun_out/band_unf $CMD > gpurun_out/band_ncu2.log 2>&1
tail -3 gpurun_out/band_ncu.log
