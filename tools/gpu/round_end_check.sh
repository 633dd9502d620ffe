# usage (on the GPU box, from the repo root): bash tools/gpu/round_end_check.sh TAG [ncu]
T=${1:-r2}
python -m pytest tests -m gpu -q --timeout 900 > gpurun_out/gpu_tests_$T.log 2>&1
timeout 1800 python bench.py > gpurun_out/bench_$T.json 2> gpurun_out/bench_$T.err
if [ "$2" = "ncu" ]; then
  B="python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-sweep --no-fp32 --no-configs"
  $B > gpurun_out/plain_$T.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_$T.csv $B > gpurun_out/ncu_launch_$T.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:vm_warp -s 3 -c 1 -o gpurun_out/prof_$T $B > gpurun_out/ncu_full_$T.log 2>&1
fi
tail -3 gpurun_out/gpu_tests_$T.log
