# ncu --set full of the store-only forward probe (bottleneck analysis).
set -e
mkdir -p gpurun_out/probe
for m in 32; do
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -DDGNN_WS_PROBE=$m scripts/ws_probe.cu \
    -Lpaper_2109_07893_b200 -ldgnn_b200 -Xlinker -rpath=$PWD/paper_2109_07893_b200 -o gpurun_out/probe/p$m
done
timeout 60 gpurun_out/probe/p32 64
ncu --set full --clock-control none --import-source on -k regex:lstm_fwd_ws -s 3 -c 1 -o gpurun_out/probe32 gpurun_out/probe/p32 64 > gpurun_out/probe_ncu.log 2>&1; echo ncu rc=$?
