bash tools/ab_wl.sh c3 "--c3-docs 200000" default hdt256 djs128 djs512 jpc512 > gpurun_out/misc_ab.log 2>&1
bash tools/ab_wl.sh c5 "" default twg8 >> gpurun_out/misc_ab.log 2>&1
cat gpurun_out/misc_ab.log
