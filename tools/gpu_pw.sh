B="python bench.py --steps 10 --warmup 3 --no-cpu-baseline"
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "f4 or seed" > gpurun_out/pw_pytest.log 2>&1; tail -1 gpurun_out/pw_pytest.log
timeout 300 $B > gpurun_out/pw_c2.log 2>&1
timeout 400 $B --config c3 > gpurun_out/pw_c3.log 2>&1
timeout 400 $B --config c5 --nq 1024 > gpurun_out/pw_c5q1024.log 2>&1
timeout 300 $B --algo tc > gpurun_out/pw_c2tc.log 2>&1
for m in 0 2 7; do UQ_TC_ABLATE=$m timeout 300 python tools/tc2_prof.py c2 > gpurun_out/pw_prof_$m.log 2>&1; done
