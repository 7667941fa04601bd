# first C3 bm_mine group: the raw metrics bench.py scales per cell (DRAM bytes, issue, FP64 pipe)
CMD3="python bench.py --workload c3 --c3-docs 100000 --steps 1 --warmup 1 --extras none --no-cpu"
M="gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__inst_executed.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active,sm__warps_active.avg.pct_of_peak_sustained_active"
ncu --metrics $M --clock-control none -k regex:"score_hits|nw_band|hits_doc|mine_ring|hits_kernel|extract_kernel" -c 40 --csv --log-file gpurun_out/r02j_c3_raw.csv $CMD3 > gpurun_out/r02j_ncu3r.log 2>&1
tail -n 2 gpurun_out/r02j_ncu3r.log; wc -l gpurun_out/r02j_c3_raw.csv
