# bench at N GPUs for several SM reserves
N=${1:-2}
mkdir -p gpurun_out
for R in 32 48 64; do
  DGNN_SM_RESERVE=$R timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port $((29600 + R)) \
    bench.py --gpus $N --steps 3 --warmup 3 --skip-cpu --skip-e2e > gpurun_out/bench_n${N}_r$R.log 2>&1
  echo -n "reserve $R: "; grep '^{' gpurun_out/bench_n${N}_r$R.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'])"
done
