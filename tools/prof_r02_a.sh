set -e
CMD="python bench.py --workload c2 --steps 1 --warmup 1 --extras none --no-cpu"
$CMD > gpurun_out/p1_plain.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:mine_ring -s 2 -c 1 -o gpurun_out/ring_c2 $CMD > gpurun_out/p1_ncu.log 2>&1
CMD3="python bench.py --workload c3 --c3-docs 100000 --steps 1 --warmup 1 --extras none --no-cpu"
$CMD3 > gpurun_out/p1_plain3.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/c3_launches.csv $CMD3 > gpurun_out/p1_ncu3.log 2>&1
