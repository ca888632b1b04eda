mkdir -p gpurun_out
CMD="python bench.py --steps 1 --warmup 1 --skip-e2e --skip-cpu"
$CMD > gpurun_out/prof_plain.log 2>&1 || { echo "plain run failed"; exit 1; }
ncu --set full --clock-control none --import-source on -k regex:"lstm_fwd_tc_kernel|lstm_bwd_tc_kernel|gcn_fwd_kernel|tn_partial_kernel" \
    -s 150 -c 8 -o gpurun_out/prof_tc $CMD > gpurun_out/ncu_tc.log 2>&1; echo full rc=$?
