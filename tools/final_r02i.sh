set -e
timeout 1400 python -m pytest tests -m gpu -x -q > gpurun_out/r02i_gputests.log 2>&1 || true
tail -n 2 gpurun_out/r02i_gputests.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02i_smoke.log 2>&1
python bench.py > gpurun_out/r02i_bench.log 2>&1
python bench.py --impl reference > gpurun_out/r02i_reference.log 2>&1
CMD3="python bench.py --workload c3 --c3-docs 100000 --steps 1 --warmup 1 --extras none --no-cpu"
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02i_c3_launches.csv $CMD3 > gpurun_out/r02i_ncu3.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:"score_hits|nw_band|hits_doc|mine_ring|hits_kernel|extract_kernel" -c 12 -o gpurun_out/r02i_c3_full $CMD3 > gpurun_out/r02i_ncu3f.log 2>&1
echo done
