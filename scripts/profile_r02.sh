# ncu evidence of the final state (1 GPU): the launch list (duration + DRAM
# bytes) of one uninstrumented timed epoch of the headline config, and one
# `--set full` capture per top kernel, all inside that region.
# usage: bash scripts/profile_r02.sh [config]   -> gpurun_out/launches_<cfg>.csv, full_<cfg>_<kernel>.ncu-rep
C=${1:-c2}
mkdir -p gpurun_out
CMD="python bench.py --config $C --steps 1 --warmup 2 --skip-e2e --skip-cpu"
$CMD > gpurun_out/prof_plain_$C.log 2>&1 || { echo "plain run failed"; tail -5 gpurun_out/prof_plain_$C.log; exit 1; }
export DGNN_PROFILE_REGION=1
ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
    --clock-control none --csv --log-file gpurun_out/launches_$C.csv $CMD > gpurun_out/ncu_launch_$C.log 2>&1
echo launches rc=$?
for k in ${KERNELS-lstm_bwd_ws_kernel lstm_dw_tc_kernel lstm_fwd_ws_kernel gcn_fwd_tc_kernel gcn_dw_tc_kernel}; do
  ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:$k -c 1 \
      -o gpurun_out/full_${C}_$k $CMD > gpurun_out/ncu_full_${C}_$k.log 2>&1; echo full $k rc=$?
done
