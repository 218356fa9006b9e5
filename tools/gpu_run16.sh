mkdir -p gpurun_out
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline"
timeout 300 $CMD > gpurun_out/plain16.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"scan_tc2" -s 1 -c 1 -o gpurun_out/prof_tc16 $CMD > gpurun_out/ncu16_full.log 2>&1
echo ncu_rc=$? >> gpurun_out/ncu16_full.log
