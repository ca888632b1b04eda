# N-GPU: NCCL parity (split-pipelined path) + bench per SM reserve / mode
N=${1:-2}
mkdir -p gpurun_out
timeout 600 python scripts/nccl_check.py --ref $N > gpurun_out/nccl_ref.log 2>&1
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29533 \
    scripts/nccl_check.py > gpurun_out/nccl_check.log 2>&1; echo nccl rc=$?; grep "OK\|differs\|Error" gpurun_out/nccl_check.log | head -3
run() {  # mode reserve
  DGNN_PIPELINED_EXCHANGE=$1 DGNN_SM_RESERVE=$2 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port $((29800 + $2)) \
    bench.py --gpus $N --steps 3 --warmup 3 --skip-cpu --skip-e2e --timeline > gpurun_out/sweep_n${N}_$1_r$2.log 2>&1
  echo -n "mode $1 reserve $2: "; grep '^{' gpurun_out/sweep_n${N}_$1_r$2.log | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step'],1), {st: (round(v['busy_ms']/3,1), round(v['idle_ms']/3,1)) for st,v in d['timeline'].items()})" || tail -5 gpurun_out/sweep_n${N}_$1_r$2.log
}
for spec in ${MODES:-auto:32 auto:16 auto:8 0:0}; do run ${spec%:*} ${spec#*:}; done
