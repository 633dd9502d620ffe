cd $GRAFT_REPO_ROOT
timeout 300 python tools/lr_probe.py 100000 100 32 256 2048 > gpurun_out/lrp.log 2>&1
timeout 300 python tools/lr_probe.py 20001 7 32 256 >> gpurun_out/lrp.log 2>&1
timeout 300 python tools/lr_probe.py 1000 25 32 256 2048 >> gpurun_out/lrp.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:vm_warp -s 1 -c 1 -o gpurun_out/prof_lrp python tools/lr_probe.py 100000 100 256 > gpurun_out/ncu_lrp.log 2>&1
cat gpurun_out/lrp.log
