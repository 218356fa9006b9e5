# summarise bench lines and tc2_prof logs given a prefix
P=$1
for f in gpurun_out/${P}_c*.log; do tail -1 $f | python -c "import json,sys; d=json.load(sys.stdin); r=d['roofline']; print('$f', d['config']['algo'], round(d['ms_per_step'],4), round(r['achieved']), round(r['frac'],3), 'scan', round(r['scan_ms_avg'],4), 'seed', round(r['seed_scan']['ms_avg'],4))" 2>/dev/null || tail -3 $f; done
for f in gpurun_out/${P}_prof_*.log; do python -c "
import json; d=json.load(open('$f')); ks=['mma_wait_tempty_frac','mma_wait_full_frac','prod_wait_empty_frac','epi_wait_tfull_frac','epi_filter_frac','mma_loop_cycles_per_item']; print('$f', {k:round(d[k],3) for k in ks}); print('   hist', {k:round(d['hist'][k],3) for k in ['mma_loop_cycles_per_item','mma_wait_tempty_frac','prod_wait_empty_frac']})" 2>/dev/null; done
