mkdir -p gpurun_out
B="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --algo asym"
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base mangled -k regex:"scan_tc2_kernelILi6ELi0ELi0E" -s 4 -c 1 -o gpurun_out/prof_asym $B > gpurun_out/pa_ncu.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"scan_tc2|merge|encode|quantize|thr_from|seed_verify" -c 80 --csv --log-file gpurun_out/pa_launches.csv $B > gpurun_out/pa_launch.log 2>&1
