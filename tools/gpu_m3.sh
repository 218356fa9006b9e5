B="python bench.py --steps 8 --warmup 3 --no-cpu-baseline"
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fuzz.py -q -x -k "search or fuzz or merge" > gpurun_out/m3_pytest.log 2>&1; tail -1 gpurun_out/m3_pytest.log
for nq in 1 4 16 32 64; do for a in popc f4; do timeout 300 $B --nq $nq --algo $a > gpurun_out/s3_${nq}_${a}.log 2>&1; done; done
timeout 300 $B --config c5 --nq 1 > gpurun_out/s3_c5q1.log 2>&1
