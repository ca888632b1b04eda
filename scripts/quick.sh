# quick GPU check: all GPU tests + one short bench line (ms, SpMM isolated / live)
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
python bench.py --steps 3 --warmup 3 --skip-cpu --skip-e2e > gpurun_out/quick.log 2>&1
grep '^{' gpurun_out/quick.log | python -c "
import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; sp=d['spmm_roofline']
print('ms', round(d['ms_per_step'],1), 'roof', r and (r['kernel'], round(r['frac'],3), round(r['frac_3xtf32_ceiling'],3), r['traffic']), 'spmm live', round(sp['frac'],3), 'isolated', round(sp['isolated']['frac'],3), round(sp['isolated']['avg_launch_us'],1))" || grep -v "^frame" gpurun_out/quick.log | tail
