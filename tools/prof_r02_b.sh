set -e
CMD="python bench.py --workload c3 --c3-docs 100000 --steps 1 --warmup 1 --extras none --no-cpu"
$CMD > gpurun_out/p2_plain.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:"score_hits|nw_band|hits_doc|extract_kernel" -c 4 -o gpurun_out/c3_banded $CMD > gpurun_out/p2_ncu.log 2>&1
