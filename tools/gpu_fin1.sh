B="python bench.py --steps 10 --warmup 3 --no-cpu-baseline"
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -q -x -k "search or full" > gpurun_out/fin1_pytest.log 2>&1; tail -1 gpurun_out/fin1_pytest.log
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base mangled -k regex:"scan_tc2_kernelILi6ELi0ELi1E" -s 2 -c 1 -o gpurun_out/prof_f4main3 $B > gpurun_out/fin1_ncu.log 2>&1
