mkdir -p gpurun_out
B="python bench.py --steps 2 --warmup 3 --no-cpu-baseline"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"scan_tc2|merge|encode|thr_from|seed_verify" -c 80 --csv --log-file gpurun_out/pf_launches_c2.csv $B > gpurun_out/pf_ncu_launch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base mangled -k regex:"scan_tc2_kernelILi6ELi0ELi1E" -s 2 -c 1 -o gpurun_out/prof_f4main2 $B > gpurun_out/pf_ncu_main.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base mangled -k regex:"scan_tc2_kernelILi6ELi1ELi1E" -s 2 -c 1 -o gpurun_out/prof_f4hist2 $B > gpurun_out/pf_ncu_hist.log 2>&1
