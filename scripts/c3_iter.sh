# graph + aggregation kernel parity, then the configs[2] and configs[1] lines at N = 1
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_kernels.py -q -x > gpurun_out/kernel_tests.log 2>&1; echo kernel tests rc=$?
tail -2 gpurun_out/kernel_tests.log
timeout 1500 python bench.py --config c3 --steps 3 --warmup 3 > gpurun_out/c3_n1.log 2>&1; echo c3 rc=$?
grep '^{' gpurun_out/c3_n1.log | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print(d['n_gpus'], round(d['ms_per_step'],1), '%.4g' % d['value'], 'e2e', d['e2e'] and round(d['e2e']['ms_per_step'],1), d['cpu_baseline'] and d['cpu_baseline']['value'])
for k,v in list(d['kernels'].items())[:10]: print('  ', k, round(v['ms_total']/d['steps'],2), v['launches']//d['steps'])" || tail -5 gpurun_out/c3_n1.log
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/c2_n1.log 2>&1; echo c2 rc=$?
grep '^{' gpurun_out/c2_n1.log | cut -c1-300
