mkdir -p gpurun_out
B="python bench.py --steps 10 --warmup 3 --no-cpu-baseline"
for sd in 32 0 128; do
  UQ_SEED_DIV=$sd timeout 300 $B > gpurun_out/b_tc_seed$sd.log 2>&1
  UQ_SEED_DIV=$sd timeout 300 $B --algo popc > gpurun_out/b_popc_seed$sd.log 2>&1
done
timeout 300 $B --config c5 --nq 1 > gpurun_out/b_c5q1.log 2>&1
timeout 300 $B --config c5 --nq 1024 > gpurun_out/b_c5q1024.log 2>&1
timeout 400 python tools/tc_ablation.py 1000000 1000 100 0 1 2 4 7 > gpurun_out/ablation.log 2>&1
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"scan_|merge_|encode_" --csv --log-file gpurun_out/launches_ours.csv $CMD > gpurun_out/ncu_list.log 2>&1; echo rc=$? >> gpurun_out/ncu_list.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"scan_tc2" -s 1 -c 1 -o gpurun_out/prof_tc_main $CMD > gpurun_out/ncu_full.log 2>&1; echo ncu_rc=$? >> gpurun_out/ncu_full.log
