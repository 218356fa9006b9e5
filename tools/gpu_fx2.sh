timeout 1200 python -m pytest tests/test_gpu_fuzz.py tests/test_gpu_parity.py -q -x -k "fuzz or f4 or seed" > gpurun_out/fx2_pytest.log 2>&1; tail -1 gpurun_out/fx2_pytest.log
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
B="python bench.py --steps 10 --warmup 3 --no-cpu-baseline"
timeout 300 $B > gpurun_out/fx2_c2.log 2>&1
timeout 400 $B --config c3 > gpurun_out/fx2_c3.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base mangled -k regex:"scan_tc2_kernelILi6ELi0ELi1E" -s 2 -c 1 -o gpurun_out/prof_f4x $B > gpurun_out/fx2_ncu.log 2>&1
