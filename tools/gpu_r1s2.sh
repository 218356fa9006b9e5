# round 1 session 2: full re-validation + bench + ncu evidence
mkdir -p gpurun_out
nvidia-smi > gpurun_out/nvsmi.txt 2>&1
(nproc; lscpu | head -20) > gpurun_out/nproc.txt
timeout 60 ./tools/peaks > gpurun_out/peaks.json 2>&1
timeout 300 python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1; echo smoke_rc=$? >> gpurun_out/smoke.log
timeout 1200 python -m pytest tests -m gpu -q --maxfail=30 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo pytest_rc=$? >> gpurun_out/pytest_gpu.log
timeout 600 python bench.py > gpurun_out/bench.log 2>&1; echo bench_rc=$? >> gpurun_out/bench.log
timeout 300 python bench.py --algo popc --no-cpu-baseline > gpurun_out/bench_popc.log 2>&1; echo rc=$? >> gpurun_out/bench_popc.log
timeout 300 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.log 2>&1; echo rc=$? >> gpurun_out/bench_ref.log
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline"
timeout 300 $CMD > gpurun_out/plain.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_list.log 2>&1
echo list_rc=$? >> gpurun_out/ncu_list.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"scan_tc" -s 2 -c 1 -o gpurun_out/prof_tc $CMD > gpurun_out/ncu_full.log 2>&1; echo ncu_rc=$? >> gpurun_out/ncu_full.log
CMDP="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --algo popc"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"scan_popc" -s 2 -c 1 -o gpurun_out/prof_popc $CMDP > gpurun_out/ncu_full_popc.log 2>&1; echo ncu_rc=$? >> gpurun_out/ncu_full_popc.log
timeout 600 ncu --set full --clock-control none -k regex:"encode_" -s 1 -c 1 -o gpurun_out/prof_enc $CMD > gpurun_out/ncu_full_enc.log 2>&1; echo ncu_rc=$? >> gpurun_out/ncu_full_enc.log
