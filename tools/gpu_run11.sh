mkdir -p gpurun_out
timeout 120 python tools/tc_sanity.py > gpurun_out/tc_sanity.log 2>&1; echo rc=$? >> gpurun_out/tc_sanity.log
timeout 500 python tools/tc_ablation.py > gpurun_out/ablation11.log 2>&1
timeout 900 python -m pytest tests -m gpu -q --maxfail=20 -p no:cacheprovider > gpurun_out/pytest_gpu11.log 2>&1; echo rc=$? >> gpurun_out/pytest_gpu11.log
