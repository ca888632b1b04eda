mkdir -p gpurun_out
CMD="python bench.py --steps 1 --warmup 1 --skip-e2e --skip-cpu"
$CMD > gpurun_out/prof_plain.log 2>&1 || { echo "plain run failed"; exit 1; }
ncu --set full --clock-control none --import-source on -k regex:"lstm_dw_tc_kernel" -s 2 -c 1 -o gpurun_out/prof_dw $CMD > gpurun_out/ncu_dw.log 2>&1; echo full rc=$?
