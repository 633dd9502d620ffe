# usage (on the GPU box): bash tools/gpu/configs_and_bench.sh [TAG] — LR gradient probes
# (specialised and interpreter), the GPU tests and the bench line
cd $GRAFT_REPO_ROOT
T=${1:-r2q}
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,temperature.gpu --format=csv > gpurun_out/smi_$T.txt
LP_CG=1 timeout 300 python tools/lr_probe.py 1000 25 32 2048 65536 > gpurun_out/lrp_$T.log 2>&1
timeout 300 python tools/lr_probe.py 1000 25 32 2048 65536 >> gpurun_out/lrp_$T.log 2>&1
LP_CG=1 timeout 300 python tools/lr_probe.py 100000 100 32 2048 >> gpurun_out/lrp_$T.log 2>&1
python -m pytest tests -m gpu -q --timeout 900 > gpurun_out/gpu_tests_$T.log 2>&1
timeout 1800 python bench.py > gpurun_out/bench_$T.json 2> gpurun_out/bench_$T.err
cat gpurun_out/lrp_$T.log; tail -3 gpurun_out/gpu_tests_$T.log
