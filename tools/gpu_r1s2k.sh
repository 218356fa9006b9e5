mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider -k "search" > gpurun_out/pytest_gpu_k.log 2>&1; echo rc=$? >> gpurun_out/pytest_gpu_k.log
B="python bench.py --steps 10 --warmup 3 --no-cpu-baseline"
timeout 300 $B > gpurun_out/b_c2_k.log 2>&1
timeout 300 $B --config c5 --nq 1024 > gpurun_out/b_c5q1024_k.log 2>&1
for m in 0 2 7 16 18 1 3; do UQ_TC_ABLATE=$m timeout 300 python tools/tc2_prof.py c2 > gpurun_out/tc2prof_k_$m.log 2>&1; done
