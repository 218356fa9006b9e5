mkdir -p gpurun_out
B="python bench.py --steps 2 --warmup 3 --no-cpu-baseline"
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base mangled -k regex:"scan_tc2_kernelILi6ELi0ELi1E" -s 2 -c 1 -o gpurun_out/prof_f4main $B > gpurun_out/f4d_ncu.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base mangled -k regex:"scan_tc2_kernelILi6ELi1ELi1E" -s 2 -c 1 -o gpurun_out/prof_f4hist $B > gpurun_out/f4d_ncu2.log 2>&1
