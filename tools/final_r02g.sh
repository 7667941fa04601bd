set -e
timeout 1400 python -m pytest tests -m gpu -x -q > gpurun_out/r02g_gputests.log 2>&1 || true
tail -2 gpurun_out/r02g_gputests.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02g_smoke.log 2>&1
python bench.py > gpurun_out/r02g2_bench.log 2>&1
CMD5="python bench.py --workload c5 --steps 1 --warmup 1 --extras none --no-cpu"
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02g_c5_launches.csv $CMD5 > gpurun_out/r02g_ncu5.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:"nw_seq" -c 1 -o gpurun_out/r02g_c5_seq $CMD5 > gpurun_out/r02g_ncu5f.log 2>&1
echo done
