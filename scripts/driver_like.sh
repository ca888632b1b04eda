# what the driver runs at round end, at N = 4 (plus N = 2 ours): reference arm first, then ours
N=${1:-4}
mkdir -p gpurun_out
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29811 \
    bench.py --impl reference --gpus $N --steps 2 --warmup 1 > gpurun_out/drv_ref_n$N.log 2>&1; echo ref rc=$?
grep '^{' gpurun_out/drv_ref_n$N.log | cut -c1-200
timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29812 \
    bench.py --gpus $N > gpurun_out/drv_n$N.log 2>&1; echo ours rc=$?
grep '^{' gpurun_out/drv_n$N.log | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('N', d['n_gpus'], 'ms', round(d['ms_per_step'],1), 'e2e', d['e2e'] and round(d['e2e']['ms_per_step'],1), 'roof', d['roofline'] and round(d['roofline']['frac'],3), d['clocks'])" || grep -v "^frame" gpurun_out/drv_n$N.log | tail -8
