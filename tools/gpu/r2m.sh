cd $GRAFT_REPO_ROOT
T=r2m
timeout 300 python tools/lr_probe.py 100000 100 32 256 2048 > gpurun_out/lrp_$T.log 2>&1
timeout 300 python tools/lr_probe.py 20001 7 32 256 >> gpurun_out/lrp_$T.log 2>&1
timeout 300 python tools/lr_probe.py 1000 25 32 256 2048 >> gpurun_out/lrp_$T.log 2>&1
for c in "config4 4096" "config3 65536" "config5 16384"; do timeout 300 python tools/config_point.py $c >> gpurun_out/lrp_$T.log 2>&1; done
S="--section SpeedOfLight --section MemoryWorkloadAnalysis --section WarpStateStats --section SchedulerStats --section Occupancy --section LaunchStats --section ComputeWorkloadAnalysis"
timeout 600 ncu $S --clock-control none -k regex:vm_warp -s 1 -c 1 -o /tmp/p_lr python tools/lr_probe.py 100000 100 256 > /dev/null 2>&1; ncu -i /tmp/p_lr.ncu-rep --page details --csv > gpurun_out/ncu_lr_$T.csv 2>&1
timeout 900 ncu $S --clock-control none -k regex:vm_warp -s 1 -c 1 -o /tmp/p_c5 python tools/config_point.py config5 16384 > /dev/null 2>&1; ncu -i /tmp/p_c5.ncu-rep --page details --csv > gpurun_out/ncu_c5_$T.csv 2>&1
timeout 900 ncu $S --clock-control none -k regex:vm_warp -s 1 -c 1 -o /tmp/p_c3 python tools/config_point.py config3 65536 > /dev/null 2>&1; ncu -i /tmp/p_c3.ncu-rep --page details --csv > gpurun_out/ncu_c3_$T.csv 2>&1
python -m pytest tests -m gpu -q --timeout 900 -x > gpurun_out/gpu_tests_$T.log 2>&1
cat gpurun_out/lrp_$T.log; tail -5 gpurun_out/gpu_tests_$T.log
