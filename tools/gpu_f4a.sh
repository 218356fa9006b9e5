mkdir -p gpurun_out
B="python bench.py --steps 10 --warmup 3 --no-cpu-baseline"
timeout 300 $B > gpurun_out/f4_b_c2_auto.log 2>&1
timeout 300 $B --algo tc > gpurun_out/f4_b_c2_tc.log 2>&1
timeout 400 $B --config c3 > gpurun_out/f4_b_c3_auto.log 2>&1
timeout 300 $B --config c5 --nq 1024 > gpurun_out/f4_b_c5q1024.log 2>&1
for m in 0 1 2 3; do UQ_TC_ABLATE=$m timeout 300 python tools/tc2_prof.py c2 > gpurun_out/f4_prof_$m.log 2>&1; done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"scan_tc2|merge|encode|thr_from" -c 60 --csv --log-file gpurun_out/f4_launches_c2.csv $B > gpurun_out/f4_ncu_launch.log 2>&1
