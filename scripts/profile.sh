# ncu evidence for the current kernels (run under gpurun, 1 GPU).
# 1) the per-launch duration list of one whole timed epoch, 2) one
# `--set full` capture per top kernel.  Summaries: scripts/ncu_summary.py.
mkdir -p gpurun_out
CMD="python bench.py --steps 1 --warmup 1 --skip-e2e --skip-cpu"
$CMD > gpurun_out/prof_plain.log 2>&1 || { echo "plain run failed"; exit 1; }
N=$(python - <<'PY'
import json
l=[x for x in open("gpurun_out/prof_plain.log") if x.startswith("{")]
print(json.loads(l[-1])["gpu_launches"])
PY
)
echo "launches per epoch: $N"
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -s $N -c $N --csv \
    --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launch.log 2>&1; echo launches rc=$?
for k in lstm_fwd_ws_kernel lstm_bwd_ws_kernel lstm_dw_tc_kernel gcn_fwd_tc_kernel gcn_dw_tc_kernel head_loss_grad_kernel; do
  ncu --set full --clock-control none --import-source on -k regex:$k -s 6 -c 1 -o gpurun_out/full_$k $CMD \
      > gpurun_out/ncu_full_$k.log 2>&1; echo full $k rc=$?
done
