B="python bench.py --steps 10 --warmup 3 --no-cpu-baseline"
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "search" > gpurun_out/ord_pytest.log 2>&1; tail -1 gpurun_out/ord_pytest.log
timeout 300 $B > gpurun_out/or_c2.log 2>&1
timeout 300 $B --algo asym > gpurun_out/or_c2asym.log 2>&1
timeout 400 $B --config c3 > gpurun_out/or_c3.log 2>&1
timeout 400 $B --config c5 --nq 1024 > gpurun_out/or_c5q1024.log 2>&1
timeout 400 $B --config c4 --n 12500000 > gpurun_out/or_c4shard.log 2>&1
timeout 900 ncu --metrics dram__bytes_read.sum,gpu__time_duration.sum --clock-control none --kernel-name-base mangled -k regex:"scan_tc2_kernelILi6ELi0ELi0E" -s 4 -c 1 python bench.py --steps 2 --warmup 3 --no-cpu-baseline --algo asym > gpurun_out/or_ncu_asym.log 2>&1
