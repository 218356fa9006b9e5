mkdir -p gpurun_out
timeout 120 python tools/tc_sanity.py > gpurun_out/tc_sanity.log 2>&1; echo rc=$? >> gpurun_out/tc_sanity.log
if grep -q "rc=0" gpurun_out/tc_sanity.log; then
  timeout 900 python -m pytest tests -m gpu -q --maxfail=20 -p no:cacheprovider > gpurun_out/pytest_gpu3.log 2>&1; echo rc=$? >> gpurun_out/pytest_gpu3.log
  timeout 300 python bench.py --steps 20 --warmup 5 > gpurun_out/bench3.log 2>&1; echo rc=$? >> gpurun_out/bench3.log
  timeout 300 python bench.py --steps 10 --warmup 3 --algo popc --no-cpu-baseline > gpurun_out/bench3_popc.log 2>&1; echo rc=$? >> gpurun_out/bench3_popc.log
  CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline"
  timeout 300 $CMD > gpurun_out/plain3.log 2>&1 && \
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"scan_|merge_|encode_" -c 40 --csv --log-file gpurun_out/launches3.csv $CMD > gpurun_out/ncu3_list.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"scan_tc" -s 1 -c 1 -o gpurun_out/prof_tc3 $CMD > gpurun_out/ncu3_full.log 2>&1
  echo ncu_rc=$? >> gpurun_out/ncu3_full.log
fi
