B="python bench.py --steps 10 --warmup 3 --no-cpu-baseline"
for dv in 8 12 16 24 32; do UQ_SEED_DIV=$dv timeout 300 $B > gpurun_out/dv_c2_$dv.log 2>&1; done
for dv in 8 16 32; do UQ_SEED_DIV=$dv timeout 300 $B --config c5 --nq 1024 > gpurun_out/dv_c5_$dv.log 2>&1; done
