B="python bench.py --steps 8 --warmup 3 --no-cpu-baseline"
for nq in 1 4 16 32 48 64 100 128 200 256 512 1000 2048 4096; do
  for a in auto popc tc f4; do
    timeout 300 $B --nq $nq --algo $a > gpurun_out/sw_${nq}_${a}.log 2>&1
    tail -1 gpurun_out/sw_${nq}_${a}.log | python -c "import json,sys
try:
  d=json.load(sys.stdin); print(json.dumps({'nq': $nq, 'algo_req': '$a', 'algo': d['config']['algo'], 'ms_per_step': d['ms_per_step'], 'value': d['value'], 'e2e': d['e2e']['value'], 'scan_ms': d['roofline']['scan_ms_avg'], 'frac': d['roofline']['frac'], 'bound': d['roofline']['bound']}))
except Exception as e: print(json.dumps({'nq': $nq, 'algo_req': '$a', 'error': 'unsupported or failed'}))" >> gpurun_out/batch_sweep.jsonl
  done
done
