bash tools/ab_wl.sh c3 "--c3-docs 200000" default nw16 nw13 default nw16 > gpurun_out/nwocc_ab.log 2>&1
cat gpurun_out/nwocc_ab.log
