bash tools/ab_wl.sh c2 "" default je2k1k je2k512 je1k1k je1k256 > gpurun_out/join_ab.log 2>&1
bash tools/ab_wl.sh c3 "--c3-docs 200000" default je2k1k >> gpurun_out/join_ab.log 2>&1
cat gpurun_out/join_ab.log
