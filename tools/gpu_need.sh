B="python bench.py --steps 10 --warmup 3 --no-cpu-baseline"
for c in 3.6 3.2 2.6 2.0; do UQ_SEED_OPT=$c timeout 300 $B > gpurun_out/nd_c2_$c.log 2>&1; done
timeout 300 $B > gpurun_out/nd_c2_def.log 2>&1
