# instruction counts / issue / duration of selected kernels: tools/ncu_kern.sh REGEX "BENCH ARGS"
M=smsp__inst_executed.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,gpu__time_duration.sum,sm__warps_active.avg.per_cycle_active
CMD="python bench.py $2 --steps 1 --warmup 1 --extras none --no-cpu"
$CMD > /dev/null 2>&1 && ncu --metrics $M --clock-control none -k regex:"$1" -c ${3:-12} --csv $CMD 2>/dev/null | grep -E '"(smsp|gpu|sm)__' | awk -F'","' '{print $5, $(NF-2), $NF}' | sed 's/(.*)//' 
