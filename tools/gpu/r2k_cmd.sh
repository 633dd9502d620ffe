cd $GRAFT_REPO_ROOT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi_r2k.txt
timeout 300 python tools/config_point.py config4 256 > gpurun_out/c4_r2k.log 2>&1
timeout 300 python tools/config_point.py config4 4096 >> gpurun_out/c4_r2k.log 2>&1
timeout 300 python tools/config_point.py config5 65536 >> gpurun_out/c4_r2k.log 2>&1
timeout 300 python tools/config_point.py config3 65536 >> gpurun_out/c4_r2k.log 2>&1
bash tools/gpu/round_end_check.sh r2k
