# multi-process parity (peer pushes and NCCL transports) vs emulated ranks at N GPUs
N=${1:-2}
mkdir -p gpurun_out
timeout 900 python scripts/nccl_check.py --ref $N > gpurun_out/nccl_ref_$N.log 2>&1; echo ref rc=$?; tail -3 gpurun_out/nccl_ref_$N.log
for tr in peer nccl; do
  DGNN_EXCHANGE=$tr timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 \
      --master-port 2971$N scripts/nccl_check.py > gpurun_out/nccl_check_${N}_$tr.log 2>&1; echo $tr rc=$?
  grep "OK\|differs\|Error\|rank 0" gpurun_out/nccl_check_${N}_$tr.log | head -8
done
