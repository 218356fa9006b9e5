set -x
mkdir -p gpurun_out
nvidia-smi > gpurun_out/nvsmi.txt 2>&1
nproc > gpurun_out/nproc.txt; lscpu | head -20 >> gpurun_out/nproc.txt
./tools/peaks > gpurun_out/peaks.json 2>&1
timeout 300 python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1
echo smoke_rc=$? >> gpurun_out/smoke.log
timeout 1200 python -m pytest tests -m gpu -q --maxfail=30 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1
echo pytest_rc=$? >> gpurun_out/pytest_gpu.log
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/bench.log 2>&1
echo bench_rc=$? >> gpurun_out/bench.log
