# round-2 C4 profile: launch list + ncu --set full of nw_band_kernel and the band-parallel extraction
CMD4="python bench.py --workload c4 --steps 1 --warmup 1 --extras none --no-cpu"
$CMD4 > gpurun_out/r02_p4c.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02_c4_launches_c.csv $CMD4 > gpurun_out/r02_ncu4c.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:"nw_band|band_exit|band_walk|score_hits|hits_doc" -c 6 -o gpurun_out/r02_c4_full $CMD4 > gpurun_out/r02_ncu4f.log 2>&1
echo done
