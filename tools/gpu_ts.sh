B="python bench.py --steps 10 --warmup 3 --no-cpu-baseline"
for t in 1e9 32 16 10; do UQ_SEED_TOPSIG=$t timeout 300 $B > gpurun_out/ts_c2_$t.log 2>&1; UQ_SEED_TOPSIG=$t timeout 300 $B --config c3 > gpurun_out/ts_c3_$t.log 2>&1; UQ_SEED_TOPSIG=$t timeout 300 $B --algo asym > gpurun_out/ts_c2asym_$t.log 2>&1; done
