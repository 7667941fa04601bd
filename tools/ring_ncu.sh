CMD="python bench.py --workload c2 --steps 1 --warmup 1 --extras none --no-cpu"
$CMD > gpurun_out/ring_p.log 2>&1 || exit 1
ncu --set full --import-source on --clock-control none -k regex:"mine_ring|hits_kernel" -s 4 -c 2 -o gpurun_out/ring_full $CMD > gpurun_out/ring_ncu.log 2>&1
tail -2 gpurun_out/ring_ncu.log
