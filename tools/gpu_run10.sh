mkdir -p gpurun_out
timeout 120 ./tools/mma_bench > gpurun_out/mma_bench2.log 2>&1
timeout 500 python tools/tc_ablation.py > gpurun_out/ablation10.log 2>&1
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline"
timeout 300 $CMD > gpurun_out/plain10.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"scan_tc2" -s 1 -c 1 -o gpurun_out/prof_tc10 $CMD > gpurun_out/ncu10_full.log 2>&1
echo ncu_rc=$? >> gpurun_out/ncu10_full.log
