python -m pytest tests -m gpu -q --timeout 900 > gpurun_out/gpu_tests_r2j.log 2>&1
timeout 1500 python bench.py > gpurun_out/bench_r2j.json 2> gpurun_out/bench_r2j.err
B="python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-sweep --no-fp32 --no-configs"
$B > gpurun_out/plain_r2j.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_r2j.csv $B > gpurun_out/ncu_launch_r2j.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:vm_warp -s 3 -c 1 -o gpurun_out/prof_r2j $B > gpurun_out/ncu_full_r2j.log 2>&1
tail -3 gpurun_out/gpu_tests_r2j.log
