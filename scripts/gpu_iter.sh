# quick iteration: selected GPU tests + short bench (no cpu / e2e legs)
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "${TESTS:-gpu}" > gpurun_out/iter_pytest.log 2>&1; echo pytest rc=$?
tail -15 gpurun_out/iter_pytest.log
timeout 600 python bench.py --steps 3 --warmup 3 --skip-cpu --skip-e2e > gpurun_out/iter_bench.log 2>&1; echo bench rc=$?
grep '^{' gpurun_out/iter_bench.log | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('ms', d['ms_per_step'], 'spmm', d['spmm_roofline'] and d['spmm_roofline']['frac'])
for k,v in d['kernels'].items(): print(k, round(v['ms_total']/d['steps'],2), v['launches'])"
