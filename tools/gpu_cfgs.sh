mkdir -p gpurun_out
B="python bench.py --steps 10 --warmup 3 --no-cpu-baseline"
P=${1:-cf}
timeout 300 $B > gpurun_out/${P}_c2.log 2>&1
timeout 400 $B --config c3 > gpurun_out/${P}_c3.log 2>&1
timeout 400 $B --config c5 --nq 1024 > gpurun_out/${P}_c5q1024.log 2>&1
timeout 400 $B --config c5 --nq 1 > gpurun_out/${P}_c5q1.log 2>&1
timeout 400 $B --config c4 --n 12500000 > gpurun_out/${P}_c4shard.log 2>&1
timeout 300 $B --config c1 > gpurun_out/${P}_c1.log 2>&1
