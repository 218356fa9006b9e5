B="python bench.py --steps 6 --warmup 3 --no-cpu-baseline --config c4 --n 12500000"
for c in 4096 2048 1024; do UQ_SEED_CAPK=$c timeout 400 $B > gpurun_out/ck_c4_$c.log 2>&1; done
