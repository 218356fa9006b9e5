mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/pytest_gpu_c.log 2>&1; echo rc=$? >> gpurun_out/pytest_gpu_c.log
timeout 600 python tools/enc_bench.py > gpurun_out/enc_bench_c.log 2>&1; echo rc=$? >> gpurun_out/enc_bench_c.log
B="python bench.py --steps 10 --warmup 3 --no-cpu-baseline"
timeout 300 $B > gpurun_out/b_c2_c.log 2>&1
timeout 300 $B --config c5 --nq 1 > gpurun_out/b_c5q1_c.log 2>&1
timeout 300 $B --config c5 --nq 1024 > gpurun_out/b_c5q1024_c.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"scan_|merge_|encode_" --csv --log-file gpurun_out/launches_c.csv $B --steps 2 > gpurun_out/ncu_list_c.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"encode_" -s 1 -c 1 -o gpurun_out/prof_enc_c $B --steps 2 > gpurun_out/ncu_enc_c.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"merge_" -s 1 -c 1 -o gpurun_out/prof_merge_c $B --steps 2 > gpurun_out/ncu_merge_c.log 2>&1
