B="python bench.py --steps 10 --warmup 3 --no-cpu-baseline --f4-index"
timeout 300 $B > gpurun_out/fx_c2.log 2>&1
timeout 400 $B --config c3 > gpurun_out/fx_c3.log 2>&1
timeout 400 $B --config c5 --nq 1024 > gpurun_out/fx_c5q1024.log 2>&1
timeout 400 $B --config c4 --n 12500000 > gpurun_out/fx_c4shard.log 2>&1
