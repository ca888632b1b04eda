# ncu full captures of the K5 variants in the isolated probe (one launch each, kx=128 hp=64, no cache)
mkdir -p gpurun_out
CMD="python scripts/lstm_probe.py --kx 128"
$CMD > gpurun_out/probe_plain.log 2>&1 || { echo "plain run failed"; exit 1; }
for k in lstm_fwd_ws_kernel lstm_fwd_pair_kernel; do
  ncu --set full --clock-control none --import-source on -k regex:$k -s 3 -c 1 -o gpurun_out/prof_$k $CMD > gpurun_out/ncu_$k.log 2>&1; echo $k rc=$?
done
