# round-2 final profiles: bench line, C3 launch list + ncu --set full (first group), C2 ring capture
set -e
python bench.py > gpurun_out/r02f_bench.log 2>&1
python bench.py --impl reference > gpurun_out/r02f_reference.log 2>&1
CMD3="python bench.py --workload c3 --c3-docs 100000 --steps 1 --warmup 1 --extras none --no-cpu"
$CMD3 > gpurun_out/r02f_p3.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02f_c3_launches.csv $CMD3 > gpurun_out/r02f_ncu3.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:"score_hits|nw_band|hits_doc|mine_ring|hits_kernel|extract_kernel" -c 10 -o gpurun_out/r02f_c3_full $CMD3 > gpurun_out/r02f_ncu3f.log 2>&1
CMD2="python bench.py --workload c2 --steps 1 --warmup 1 --extras none --no-cpu"
$CMD2 > gpurun_out/r02f_p2.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02f_c2_launches.csv $CMD2 > gpurun_out/r02f_ncu2.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:"mine_ring|hits_kernel" -s 4 -c 2 -o gpurun_out/r02f_c2_full $CMD2 > gpurun_out/r02f_ncu2f.log 2>&1
CMD5="python bench.py --workload c5 --steps 1 --warmup 1 --extras none --no-cpu"
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02f_c5_launches.csv $CMD5 > gpurun_out/r02f_ncu5.log 2>&1
echo done
