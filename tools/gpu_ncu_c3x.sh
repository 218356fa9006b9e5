B="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --config c3 --n 2000000 --nq 2048"
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base mangled -k regex:"scan_tc2_kernelILi8ELi0ELi1E" -s 2 -c 1 -o gpurun_out/prof_c3x $B > gpurun_out/c3x_ncu.log 2>&1
tail -1 gpurun_out/c3x_ncu.log
