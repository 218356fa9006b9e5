B="python bench.py --steps 10 --warmup 3 --no-cpu-baseline"
UQ_TC2_S=37 timeout 300 $B > gpurun_out/un_c2_37.log 2>&1
UQ_TC2_S=37 timeout 900 ncu --metrics dram__bytes_read.sum,gpu__time_duration.sum --clock-control none --kernel-name-base mangled -k regex:"scan_tc2_kernelILi6ELi0ELi1E" -s 4 -c 1 $B > gpurun_out/un_ncu37.log 2>&1
UQ_TC2_UNIFORM=1 timeout 300 $B > gpurun_out/un_c2_1b.log 2>&1
timeout 300 $B > gpurun_out/un_c2_0b.log 2>&1
