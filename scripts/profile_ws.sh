mkdir -p gpurun_out
CMD="python bench.py --steps 1 --warmup 1 --skip-e2e --skip-cpu"
$CMD > gpurun_out/prof_plain.log 2>&1 || { echo "plain run failed"; exit 1; }
ncu --set full --clock-control none --import-source on -k regex:"lstm_fwd_ws_kernel|lstm_bwd_ws_kernel|lstm_dw_tc_kernel" \
    -s 40 -c 5 -o gpurun_out/prof_ws $CMD > gpurun_out/ncu_ws.log 2>&1; echo full rc=$?
