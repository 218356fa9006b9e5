B="python bench.py --steps 10 --warmup 3 --no-cpu-baseline"
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "f4_index" 2>&1 | tail -1
timeout 300 $B > gpurun_out/l2_c2.log 2>&1
timeout 400 $B --config c5 --nq 1024 > gpurun_out/l2_c5q1024.log 2>&1
timeout 400 $B --config c3 > gpurun_out/l2_c3.log 2>&1
timeout 900 ncu --metrics dram__bytes_read.sum,gpu__time_duration.sum --clock-control none --kernel-name-base mangled -k regex:"scan_tc2_kernelILi6ELi0ELi1E" -s 2 -c 1 $B > gpurun_out/l2_ncu.log 2>&1
grep -E "dram__bytes|gpu__time" gpurun_out/l2_ncu.log
