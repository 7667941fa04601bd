CMD3="python bench.py --workload c3 --c3-docs 100000 --steps 1 --warmup 1 --extras none --no-cpu"
ncu --set full --import-source on --clock-control none -k regex:"score_hits|nw_band|hits_doc|extract_kernel" -c 4 -o gpurun_out/r02i_c3_banded $CMD3 > gpurun_out/r02i_ncu3b.log 2>&1
tail -n 2 gpurun_out/r02i_ncu3b.log
