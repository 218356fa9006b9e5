mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider --durations=15 > gpurun_out/pytest_gpu_m.log 2>&1; echo rc=$? >> gpurun_out/pytest_gpu_m.log
B="python bench.py --steps 10 --warmup 3 --no-cpu-baseline"
timeout 300 $B > gpurun_out/b_c2_m.log 2>&1
timeout 300 $B --config c1 > gpurun_out/b_c1_m.log 2>&1
