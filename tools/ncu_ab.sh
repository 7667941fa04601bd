# instruction counts / issue / duration of the ring kernel per variant (C2)
M=smsp__inst_executed.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,gpu__time_duration.sum,smsp__warps_issue_stalled_wait.avg,smsp__warps_issue_stalled_long_scoreboard.avg,smsp__warps_issue_stalled_barrier.avg,smsp__warps_issue_stalled_short_scoreboard.avg,smsp__warps_issue_stalled_math_pipe_throttle.avg,smsp__warps_issue_stalled_no_instruction.avg,smsp__warps_issue_stalled_sleeping.avg,smsp__warps_active.avg
for v in "$@"; do
  if [ "$v" = "default" ]; then unset BM_LIB_PATH; else export BM_LIB_PATH=tools/_prof/$v.so; fi
  CMD="python bench.py --workload c2 --steps 1 --warmup 1 --extras none --no-cpu"
  $CMD > /dev/null 2>&1 && ncu --metrics $M --clock-control none -k regex:mine_ring -s 2 -c 1 --csv $CMD 2>/dev/null | grep -E '"(smsp|gpu)__' | awk -F'","' -v v=$v '{print v, $(NF-2), $NF}'
done
