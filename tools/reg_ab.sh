bash tools/ab_wl.sh c5 "" default base_r02 > gpurun_out/reg_ab.log 2>&1
bash tools/ab_wl.sh c3 "--c3-docs 200000" default base_r02 >> gpurun_out/reg_ab.log 2>&1
bash tools/ab_wl.sh c2 "" default base_r02 >> gpurun_out/reg_ab.log 2>&1
cat gpurun_out/reg_ab.log
