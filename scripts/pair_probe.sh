# Build + run the CTA-pair forward-kernel bottleneck probe for several masks (GPU box).
set -e
mkdir -p gpurun_out/probe
MASKS="0 1 2 4 8 16 9 14 6 12"
for m in $MASKS; do
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -DDGNN_PAIR_PROBE=$m scripts/pair_probe.cu \
    -Lpaper_2109_07893_b200 -ldgnn_b200 -Xlinker -rpath=$PWD/paper_2109_07893_b200 -o gpurun_out/probe/pp$m &
done
wait
for m in $MASKS; do timeout 60 gpurun_out/probe/pp$m 128; done
