mkdir -p gpurun_out
timeout 600 python tools/tc_ablation.py > gpurun_out/ablation5.log 2>&1
timeout 600 python tools/tc_ablation.py 1000000 128 100 >> gpurun_out/ablation5.log 2>&1
