B="python bench.py --steps 10 --warmup 3 --no-cpu-baseline"
for fm in 4 2.5 1.7; do UQ_SEED_FLOORMULT=$fm timeout 300 $B > gpurun_out/fm_c2_$fm.log 2>&1; UQ_SEED_FLOORMULT=$fm timeout 300 $B --config c5 --nq 1024 > gpurun_out/fm_c5_$fm.log 2>&1; done
UQ_SEED_FLOORMULT=2.5 timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "seed" > gpurun_out/fm_pytest.log 2>&1; tail -1 gpurun_out/fm_pytest.log
