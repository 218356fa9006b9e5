mkdir -p gpurun_out
timeout 300 python __graft_entry__.py smoke > gpurun_out/smoke_f.log 2>&1; echo smoke_rc=$? >> gpurun_out/smoke_f.log
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider --durations=10 > gpurun_out/pytest_gpu_f.log 2>&1; echo rc=$? >> gpurun_out/pytest_gpu_f.log
timeout 600 python bench.py > gpurun_out/bench_f.log 2>&1; echo rc=$? >> gpurun_out/bench_f.log
timeout 300 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref_f.log 2>&1
