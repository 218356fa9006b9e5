mkdir -p gpurun_out
B="python bench.py --steps 10 --warmup 3 --no-cpu-baseline"
for c in 0 4 2; do UQ_SEED_OPT=$c timeout 300 $B > gpurun_out/f4f_c2_opt$c.log 2>&1; UQ_SEED_OPT=$c timeout 300 python tools/tc2_prof.py c2 > gpurun_out/f4f_prof_opt$c.log 2>&1; done
