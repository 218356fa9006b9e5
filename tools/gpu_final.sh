mkdir -p gpurun_out
timeout 2000 python -m pytest tests -q -m gpu -p no:cacheprovider > gpurun_out/final_pytest.log 2>&1; tail -3 gpurun_out/final_pytest.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final_smoke.log 2>&1; tail -1 gpurun_out/final_smoke.log
timeout 600 python bench.py > gpurun_out/final_bench_c2.log 2>&1
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/final_bench_ref.log 2>&1
bash tools/gpu_cfgs.sh fc
B="python bench.py --steps 10 --warmup 3 --no-cpu-baseline"
timeout 300 $B --algo asym > gpurun_out/fc_c2asym.log 2>&1
timeout 300 $B --algo tc > gpurun_out/fc_c2tc.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"scan_tc2|merge|encode|thr_from|seed_verify" -c 80 --csv --log-file gpurun_out/fc_launches_c2.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/fc_ncu_launch.log 2>&1
