bash tools/ab_wl.sh c3 "--c3-docs 200000" sm5 sm6 sm8 sm5 sm6 > gpurun_out/sm_ab2.log 2>&1
bash tools/ab_wl.sh c4 "" default sm5 sm6 >> gpurun_out/sm_ab2.log 2>&1
cat gpurun_out/sm_ab2.log
