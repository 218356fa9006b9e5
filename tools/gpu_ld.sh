B="python bench.py --steps 10 --warmup 3 --no-cpu-baseline"
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "search" > gpurun_out/ld_pytest.log 2>&1; tail -1 gpurun_out/ld_pytest.log
timeout 300 $B > gpurun_out/ld_c2.log 2>&1
timeout 400 $B --config c3 > gpurun_out/ld_c3.log 2>&1
timeout 400 $B --config c5 --nq 1024 > gpurun_out/ld_c5q1024.log 2>&1
timeout 400 $B --config c4 --n 12500000 > gpurun_out/ld_c4shard.log 2>&1
timeout 300 $B --algo tc > gpurun_out/ld_c2tc.log 2>&1
