timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "asym or f4_index" > gpurun_out/i8x_pytest.log 2>&1; tail -1 gpurun_out/i8x_pytest.log
B="python bench.py --steps 10 --warmup 3 --no-cpu-baseline --algo asym"
timeout 300 $B > gpurun_out/ix_c2asym.log 2>&1
timeout 400 $B --config c3 > gpurun_out/ix_c3asym.log 2>&1
