mkdir -p gpurun_out
timeout 120 python tools/tc_sanity.py > gpurun_out/tc_sanity.log 2>&1; echo rc=$? >> gpurun_out/tc_sanity.log
./tools/peaks > gpurun_out/peaks2.json 2>&1
if grep -q "rc=0" gpurun_out/tc_sanity.log; then
  timeout 900 python -m pytest tests -m gpu -q --maxfail=20 -p no:cacheprovider > gpurun_out/pytest_gpu2.log 2>&1; echo rc=$? >> gpurun_out/pytest_gpu2.log
  timeout 300 python bench.py --steps 10 --warmup 3 --algo tc --no-cpu-baseline > gpurun_out/bench_tc.log 2>&1; echo rc=$? >> gpurun_out/bench_tc.log
fi
