# round-2 final C3 capture: every kernel of the first bm_mine group (-c 13 covers the fused tier's
# four hits/ring pairs, hits_doc, score_hits, nw_band, extract and the next group's first kernel)
CMD3="python bench.py --workload c3 --c3-docs 100000 --steps 1 --warmup 1 --extras none --no-cpu"
ncu --set full --import-source on --clock-control none -k regex:"score_hits|nw_band|hits_doc|mine_ring|hits_kernel|extract_kernel" -c 13 -o gpurun_out/r02f_c3_full13 $CMD3 > gpurun_out/r02f_ncu3g.log 2>&1
echo done
