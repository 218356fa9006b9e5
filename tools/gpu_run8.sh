mkdir -p gpurun_out
timeout 120 python tools/tc_sanity.py > gpurun_out/tc_sanity.log 2>&1; echo rc=$? >> gpurun_out/tc_sanity.log
timeout 900 python -m pytest tests -m gpu -q --maxfail=20 -p no:cacheprovider > gpurun_out/pytest_gpu8.log 2>&1; echo rc=$? >> gpurun_out/pytest_gpu8.log
timeout 500 python tools/tc_ablation.py > gpurun_out/ablation8.log 2>&1
timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench8.log 2>&1; echo rc=$? >> gpurun_out/bench8.log
timeout 300 python bench.py --steps 10 --warmup 3 --algo popc --no-cpu-baseline > gpurun_out/bench8_popc.log 2>&1; echo rc=$? >> gpurun_out/bench8_popc.log
