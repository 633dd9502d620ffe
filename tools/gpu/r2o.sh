cd $GRAFT_REPO_ROOT
T=r2o
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,temperature.gpu --format=csv > gpurun_out/smi_$T.txt
timeout 300 python tools/lr_probe.py 100000 100 32 2048 > gpurun_out/lrp_$T.log 2>&1
timeout 300 python tools/lr_probe.py 1000 25 32 2048 65536 >> gpurun_out/lrp_$T.log 2>&1
LP_CG=1 timeout 300 python tools/lr_probe.py 100000 100 32 2048 >> gpurun_out/lrp_$T.log 2>&1
python -m pytest tests -m gpu -q --timeout 900 > gpurun_out/gpu_tests_$T.log 2>&1
timeout 1800 python bench.py > gpurun_out/bench_$T.json 2> gpurun_out/bench_$T.err
B="python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-sweep --no-fp32 --no-configs"
$B > gpurun_out/plain_$T.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_$T.csv $B > gpurun_out/ncu_launch_$T.log 2>&1
ncu --set full --clock-control none -k regex:vm_warp -s 3 -c 1 -o /tmp/prof_$T $B > gpurun_out/ncu_full_$T.log 2>&1
ncu -i /tmp/prof_$T.ncu-rep --page details --csv > gpurun_out/ncu_details_$T.csv 2>&1
ncu -i /tmp/prof_$T.ncu-rep --page raw --csv > gpurun_out/ncu_raw_$T.csv 2>&1
ls -la /tmp/prof_$T.ncu-rep
cat gpurun_out/lrp_$T.log; tail -3 gpurun_out/gpu_tests_$T.log
