# A/B of the index-fed top-k epilogue: pipelined TMEM loads (libuq.so) vs the plain loop (libuq_ab_nopipe.so, -DUQ_EPI_PIPE=0)
run() { python bench.py --config $1 $3 --steps 10 --no-extras --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); r=d['roofline']; print('$1 $2', round(r['scan_ms_avg'],4), round(r['frac'],3), d['clocks']['sm_mhz'], d['digest']['all'][:8])"; }
for i in 1 2; do
  run c2 pipe ""; UQ_LIB_AB=$PWD/paper_2506_00528_b200/libuq_ab_nopipe.so run c2 nopipe ""
  run c3 pipe "--x 256"; UQ_LIB_AB=$PWD/paper_2506_00528_b200/libuq_ab_nopipe.so run c3 nopipe "--x 256"
  run c5 pipe "--queries 1024"; UQ_LIB_AB=$PWD/paper_2506_00528_b200/libuq_ab_nopipe.so run c5 nopipe "--queries 1024"
done
