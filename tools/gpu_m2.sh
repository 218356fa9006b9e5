B="python bench.py --steps 8 --warmup 3 --no-cpu-baseline"
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fuzz.py -q -x > gpurun_out/m2_pytest.log 2>&1; tail -1 gpurun_out/m2_pytest.log
rm -f gpurun_out/batch_sweep2.jsonl
for nq in 1 4 16 32 48 64 100 128; do
  for a in popc tc f4; do
    timeout 300 $B --nq $nq --algo $a > gpurun_out/s2_${nq}_${a}.log 2>&1
    tail -1 gpurun_out/s2_${nq}_${a}.log | python -c "import json,sys
d=json.load(sys.stdin); print(json.dumps({'nq': $nq, 'algo': d['config']['algo'], 'ms_per_step': d['ms_per_step'], 'value': d['value'], 'scan_ms': d['roofline']['scan_ms_avg']}))" >> gpurun_out/batch_sweep2.jsonl
  done
done
timeout 300 $B --config c5 --nq 1 > gpurun_out/s2_c5q1.log 2>&1
