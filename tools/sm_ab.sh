bash tools/ab_wl.sh c3 "--c3-docs 200000" default sm5 sm3 default sm5 > gpurun_out/sm_ab.log 2>&1
bash tools/ab_wl.sh c5 "" default sm5 >> gpurun_out/sm_ab.log 2>&1
cat gpurun_out/sm_ab.log
