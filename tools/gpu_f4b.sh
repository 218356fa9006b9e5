mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "search" > gpurun_out/f4b_pytest.log 2>&1; echo rc=$? >> gpurun_out/f4b_pytest.log
B="python bench.py --steps 10 --warmup 3 --no-cpu-baseline"
timeout 300 $B > gpurun_out/f4b_c2.log 2>&1
timeout 400 $B --config c3 > gpurun_out/f4b_c3.log 2>&1
for m in 0 2; do UQ_TC_ABLATE=$m timeout 300 python tools/tc2_prof.py c2 > gpurun_out/f4b_prof_$m.log 2>&1; done
