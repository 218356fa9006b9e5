mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider -k "search" > gpurun_out/pytest_gpu_j.log 2>&1; echo rc=$? >> gpurun_out/pytest_gpu_j.log
B="python bench.py --steps 10 --warmup 3 --no-cpu-baseline"
timeout 300 $B > gpurun_out/b_c2_j.log 2>&1
timeout 300 $B --config c5 --nq 1024 > gpurun_out/b_c5q1024_j.log 2>&1
timeout 300 python tools/tc2_prof.py c2 > gpurun_out/tc2prof_j.log 2>&1
UQ_TC_ABLATE=2 timeout 300 python tools/tc2_prof.py c2 > gpurun_out/tc2prof_j_abl2.log 2>&1
UQ_TC_ABLATE=7 timeout 300 python tools/tc2_prof.py c2 > gpurun_out/tc2prof_j_abl7.log 2>&1
