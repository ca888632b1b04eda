# backward LSTM step kernel (K6): dz producer warp count
set -e
mkdir -p gpurun_out/probe
V=${V:-"8 4 16"}
for p in $V; do
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 --expt-relaxed-constexpr -DDGNN_BWD_NPROD=$p scripts/bwd_probe.cu \
    -Lpaper_2109_07893_b200 -ldgnn_b200 -Xlinker -rpath=$PWD/paper_2109_07893_b200 -o gpurun_out/probe/b_$p &
done
wait
for kx in 128 64; do for p in $V; do timeout 60 gpurun_out/probe/b_$p $kx | tail -1; done; done
