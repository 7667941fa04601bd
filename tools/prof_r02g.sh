# round-2 (second session) profiles: bench line + reference arm on the final tree, C3/C2 launch
# lists, ncu --set full of the C3 first group and the C2 ring, and the opt-in fused banded tier
set -e
python bench.py > gpurun_out/r02g_bench.log 2>&1
python bench.py --impl reference > gpurun_out/r02g_reference.log 2>&1
CMD3="python bench.py --workload c3 --c3-docs 100000 --steps 1 --warmup 1 --extras none --no-cpu"
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02g_c3_launches.csv $CMD3 > gpurun_out/r02g_ncu3.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:"score_hits|nw_band|hits_doc|mine_ring|hits_kernel|extract_kernel" -c 10 -o gpurun_out/r02g_c3_full $CMD3 > gpurun_out/r02g_ncu3f.log 2>&1
BM_BAND_FUSED=1 ncu --set full --import-source on --clock-control none -k regex:"mine_band" -c 1 -o gpurun_out/r02g_c3_band $CMD3 > gpurun_out/r02g_ncu3b.log 2>&1
CMD2="python bench.py --workload c2 --steps 1 --warmup 1 --extras none --no-cpu"
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02g_c2_launches.csv $CMD2 > gpurun_out/r02g_ncu2.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:"mine_ring|hits_kernel" -s 4 -c 2 -o gpurun_out/r02g_c2_full $CMD2 > gpurun_out/r02g_ncu2f.log 2>&1
echo done
