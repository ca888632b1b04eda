# peer (copy-engine) exchange: probe, NCCL-vs-emulated parity through the peer path, bench N=2 (and N=4)
N=${1:-2}
mkdir -p gpurun_out
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29701 \
    scripts/symm_probe.py > gpurun_out/symm_probe.log 2>&1; echo probe rc=$?; grep "rank 0\|rendezvous\|Error\|error" gpurun_out/symm_probe.log | head -8
timeout 600 python scripts/nccl_check.py --ref $N > gpurun_out/nccl_ref.log 2>&1
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29702 \
    scripts/nccl_check.py > gpurun_out/nccl_check.log 2>&1; echo parity rc=$?; grep "OK\|differs\|Error\|rank 0" gpurun_out/nccl_check.log | head -4
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29703 \
    bench.py --gpus $N --steps 3 --warmup 3 --skip-cpu --skip-e2e --timeline > gpurun_out/peer_n$N.log 2>&1; echo bench rc=$?
grep '^{' gpurun_out/peer_n$N.log | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('N', d['n_gpus'], 'ms', round(d['ms_per_step'],1), {st: (round(v['busy_ms']/3,1), round(v['idle_ms']/3,1), {k: round(x/3,1) for k,x in list(v['idle_before'].items())[:4]}) for st,v in d['timeline'].items()})" || grep -v "^frame" gpurun_out/peer_n$N.log | tail -12
