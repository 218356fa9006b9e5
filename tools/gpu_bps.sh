B="python bench.py --steps 10 --warmup 3 --no-cpu-baseline"
timeout 300 $B --algo tc > gpurun_out/bi_c2tc.log 2>&1
timeout 300 $B --algo asym > gpurun_out/bi_c2asym.log 2>&1
timeout 400 $B --algo asym --config c3 > gpurun_out/bi_c3asym.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "tc or asym" > gpurun_out/bi_pytest.log 2>&1; tail -1 gpurun_out/bi_pytest.log
