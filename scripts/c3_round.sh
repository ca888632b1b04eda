# configs[2] TM-GCN line at 1 and 4 GPUs (gpurun --gpus 4)
mkdir -p gpurun_out
timeout 1500 python bench.py --config c3 --steps 3 --warmup 3 > gpurun_out/c3_n1.log 2>&1; echo n1 rc=$?
timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29640 \
    bench.py --config c3 --gpus 4 --steps 3 --warmup 3 --skip-cpu > gpurun_out/c3_n4.log 2>&1; echo n4 rc=$?
for N in 1 4; do grep '^{' gpurun_out/c3_n$N.log | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print(d['n_gpus'], round(d['ms_per_step'],1), '%.4g' % d['value'], 'e2e', d['e2e'] and round(d['e2e']['ms_per_step'],1), 'prep', round(d['prep_seconds']), d['cpu_baseline'] and d['cpu_baseline']['value'])
for k,v in list(d['kernels'].items())[:8]: print('  ', k, round(v['ms_total']/d['steps'],2), v['launches']//d['steps'])" || tail -5 gpurun_out/c3_n$N.log; done
