# per-stream idle breakdown at N=1 and N=2 (bench --timeline)
mkdir -p gpurun_out
python bench.py --steps 2 --warmup 3 --skip-cpu --skip-e2e --timeline > gpurun_out/tl_n1.log 2>&1; echo n1 rc=$?
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29534 \
    bench.py --gpus 2 --steps 2 --warmup 3 --skip-cpu --skip-e2e --timeline > gpurun_out/tl_n2.log 2>&1; echo n2 rc=$?
for f in gpurun_out/tl_n1.log gpurun_out/tl_n2.log; do
grep '^{' $f | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('N', d['n_gpus'], 'ms', d['ms_per_step'])
for st, v in d['timeline'].items(): print(' stream', st, 'busy', round(v['busy_ms']/d['steps'],1), 'idle', round(v['idle_ms']/d['steps'],1), {k: round(x/d['steps'],1) for k,x in v['idle_before'].items()})
"; done
