set -e
CMD3="python bench.py --workload c3 --c3-docs 100000 --steps 1 --warmup 1 --extras none --no-cpu"
$CMD3 > gpurun_out/r02_p3b.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:"score_hits|nw_band|hits_doc|extract_kernel" -c 4 -o gpurun_out/r02_c3_banded $CMD3 > gpurun_out/r02_ncu3b.log 2>&1
CMD4="python bench.py --workload c4 --steps 1 --warmup 1 --extras none --no-cpu"
$CMD4 > gpurun_out/r02_p4.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02_c4_launches.csv $CMD4 > gpurun_out/r02_ncu4.log 2>&1
