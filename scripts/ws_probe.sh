# Build + run the forward-kernel bottleneck probe for every mask (GPU box).
set -e
mkdir -p gpurun_out/probe
for m in 0 16 32 48; do
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -DDGNN_WS_PROBE=$m scripts/ws_probe.cu \
    -Lpaper_2109_07893_b200 -ldgnn_b200 -Xlinker -rpath=$PWD/paper_2109_07893_b200 -o gpurun_out/probe/p$m
done
for m in 0 16 32 48; do timeout 60 gpurun_out/probe/p$m 64; done
timeout 60 gpurun_out/probe/p0 128
