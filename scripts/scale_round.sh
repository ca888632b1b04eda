# bench at N = 1, 2, 4 on one box (gpurun --gpus 4)
mkdir -p gpurun_out
python bench.py --steps 5 --warmup 3 --skip-cpu > gpurun_out/scale_n1.log 2>&1; echo n1 rc=$?
for N in 2 4; do
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port $((29600+N)) \
    bench.py --gpus $N --steps 5 --warmup 3 --skip-cpu > gpurun_out/scale_n$N.log 2>&1; echo n$N rc=$?
done
for N in 1 2 4; do grep '^{' gpurun_out/scale_n$N.log | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print(d['n_gpus'], round(d['ms_per_step'],1), '%.4g' % d['value'], 'e2e', d['e2e'] and round(d['e2e']['ms_per_step'],1), d['clocks'])"; done
