B="python bench.py --steps 10 --warmup 3 --no-cpu-baseline"
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "popc" > gpurun_out/pp_pytest.log 2>&1; tail -1 gpurun_out/pp_pytest.log
timeout 400 $B --config c5 --nq 1 > gpurun_out/pp_c5q1.log 2>&1
timeout 300 $B --nq 1 > gpurun_out/pp_c2q1.log 2>&1
timeout 300 $B --nq 4 > gpurun_out/pp_c2q4.log 2>&1
timeout 300 $B --config c1 > gpurun_out/pp_c1.log 2>&1
