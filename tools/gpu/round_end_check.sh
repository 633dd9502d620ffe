# usage (on the GPU box, from the repo root): bash tools/gpu/round_end_check.sh TAG [ncu]
# GPU tests, the bench line, and (with "ncu") the launch list plus one --set full capture of
# the bench's VM launch, exported as CSV (the report itself stays in /tmp: it is large)
T=${1:-r2}
python -m pytest tests -m gpu -q --timeout 900 > gpurun_out/gpu_tests_$T.log 2>&1
timeout 1800 python bench.py > gpurun_out/bench_$T.json 2> gpurun_out/bench_$T.err
if [ "$2" = "ncu" ]; then
  B="python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-sweep --no-fp32 --no-configs"
  $B > gpurun_out/plain_$T.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_$T.csv $B > gpurun_out/ncu_launch_$T.log 2>&1
  ncu --set full --clock-control none -k regex:vm_warp -s 3 -c 1 -o /tmp/prof_$T $B > gpurun_out/ncu_full_$T.log 2>&1
  ncu -i /tmp/prof_$T.ncu-rep --page details --csv > gpurun_out/ncu_details_$T.csv 2>&1
  ncu -i /tmp/prof_$T.ncu-rep --page raw --csv > gpurun_out/ncu_raw_$T.csv 2>&1
fi
tail -3 gpurun_out/gpu_tests_$T.log
