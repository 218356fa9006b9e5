B="python bench.py --steps 10 --warmup 3 --no-cpu-baseline"
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fuzz.py -q -x -k "f4_index or fuzz" 2>&1 | tail -1
timeout 300 $B > gpurun_out/xm_c2.log 2>&1
timeout 400 $B --config c3 > gpurun_out/xm_c3.log 2>&1
timeout 400 $B --config c5 --nq 1024 > gpurun_out/xm_c5q1024.log 2>&1
timeout 400 $B --config c4 --n 12500000 > gpurun_out/xm_c4shard.log 2>&1
