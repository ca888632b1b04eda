# round-2 iteration: c2 bench line (no CPU leg) + c4 line at N=1
mkdir -p gpurun_out
#timeout 900 python bench.py --steps 3 --warmup 3 --skip-cpu > gpurun_out/r02_c2.log 2>&1; echo c2 rc=$?
#grep '^{' gpurun_out/r02_c2.log > gpurun_out/r02_c2.json || tail -20 gpurun_out/r02_c2.log
timeout 1500 python bench.py --config c4 --steps 2 --warmup 3 --skip-cpu > gpurun_out/r02_c4_n1.log 2>&1; echo c4 rc=$?
grep '^{' gpurun_out/r02_c4_n1.log > gpurun_out/r02_c4_n1.json || tail -20 gpurun_out/r02_c4_n1.log
for f in gpurun_out/r02_c4_n1.json; do python -c "
import json,sys; d=json.load(open('$f')); e=d['e2e'] or {}
print('$f', 'ms', round(d['ms_per_step'],1), 'value', '%.3g'%d['value'], 'prep', round(d['prep_seconds'],1), 'dom', d['roofline'] and (d['roofline']['kernel'], round(d['roofline']['frac'],3)), 'spmm', d['spmm_roofline'] and round(d['spmm_roofline']['frac'],3))
print('  e2e ms', e.get('ms_per_step'), 'delta', e.get('delta_vs_full_bytes'), e.get('delta_vs_full_bytes_reference_schedule'), 'pcie', e.get('pcie'))
for k,v in list(d['kernels'].items())[:12]: print('  ', k, round(v['ms_total']/d['steps'],2), v['launches']//d['steps'], v.get('hbm_frac') and round(v['hbm_frac'],3))
"; done
