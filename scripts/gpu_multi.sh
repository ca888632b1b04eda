# 2-GPU checks: NCCL parity vs emulated ranks, then the bench at N=2.
mkdir -p gpurun_out
N=${1:-2}
timeout 600 python scripts/nccl_check.py --ref $N > gpurun_out/nccl_ref.log 2>&1; echo ref rc=$?; tail -2 gpurun_out/nccl_ref.log
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29533 \
    scripts/nccl_check.py > gpurun_out/nccl_check.log 2>&1; echo nccl rc=$?; tail -6 gpurun_out/nccl_check.log
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29534 \
    bench.py --gpus $N --steps 3 --warmup 3 --skip-cpu > gpurun_out/bench_n$N.log 2>&1; echo bench rc=$?
grep '^{' gpurun_out/bench_n$N.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['n_gpus'], d['ms_per_step'], d['value'], d.get('e2e') and d['e2e']['ms_per_step'])" || tail -30 gpurun_out/bench_n$N.log
