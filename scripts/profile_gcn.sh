mkdir -p gpurun_out
CMD="python bench.py --steps 1 --warmup 1 --skip-e2e --skip-cpu"
$CMD > gpurun_out/prof_plain.log 2>&1 || { echo "plain run failed"; exit 1; }
ncu --set full --clock-control none --import-source on -k regex:gcn_fwd_tc_kernel -s 3 -c 1 -o gpurun_out/full_gcn_fwd_tc_kernel $CMD > gpurun_out/ncu_gcn.log 2>&1; echo full rc=$?
