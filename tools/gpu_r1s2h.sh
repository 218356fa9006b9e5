mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/pytest_gpu_h.log 2>&1; echo rc=$? >> gpurun_out/pytest_gpu_h.log
B="python bench.py --steps 10 --warmup 3 --no-cpu-baseline"
for sd in 8 4 16 0; do UQ_SEED_DIV=$sd timeout 300 $B > gpurun_out/b_c2_h_seed$sd.log 2>&1; done
timeout 300 $B --config c5 --nq 1024 > gpurun_out/b_c5q1024_h.log 2>&1
timeout 300 python tools/tc_ablation.py 1000000 1000 100 0 2 7 > gpurun_out/ablation_h.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"scan_|merge_|encode_|thr_" --csv --log-file gpurun_out/launches_h.csv $B --steps 2 > gpurun_out/ncu_list_h.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:"scan_tc2_kernel<6, 0>" -s 1 -c 1 -o gpurun_out/prof_tc2_main_h $B --steps 2 > gpurun_out/ncu_tc2_h.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:"scan_tc2_kernel<6, 1>" -s 1 -c 1 -o gpurun_out/prof_tc2_hist_h $B --steps 2 > gpurun_out/ncu_tc2hist_h.log 2>&1
