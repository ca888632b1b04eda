# ncu evidence for the current kernels (run under gpurun, 1 GPU)
mkdir -p gpurun_out
CMD="python bench.py --steps 1 --warmup 1 --skip-e2e --skip-cpu"
$CMD > gpurun_out/prof_plain.log 2>&1 || { echo "plain run failed"; exit 1; }
ncu --metrics gpu__time_duration.sum --clock-control none -s 3500 -c 2600 --csv \
    --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launch.log 2>&1; echo launches rc=$?
ncu --set full --clock-control none --import-source on \
    -k regex:"lstm_fwd_kernel|lstm_bwd_kernel|tn_partial_kernel|gcn_fwd_kernel|lap_write_kernel|transpose_scatter_kernel" \
    -s 60 -c 12 -o gpurun_out/prof_full $CMD > gpurun_out/ncu_full.log 2>&1; echo full rc=$?
ls -la gpurun_out
