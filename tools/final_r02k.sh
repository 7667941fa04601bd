set -e
timeout 1400 python -m pytest tests -m gpu -x -q > gpurun_out/r02k_gputests.log 2>&1 || true
tail -n 2 gpurun_out/r02k_gputests.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02k_smoke.log 2>&1
python bench.py > gpurun_out/r02k_bench.log 2>&1
python bench.py --impl reference > gpurun_out/r02k_reference.log 2>&1
echo done
