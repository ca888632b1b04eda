# K5 at hidden 32 (configs[3]/[4]): epilogue warp count
set -e
mkdir -p gpurun_out/probe
for e in 16 8; do
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 --expt-relaxed-constexpr -DHPP=32 -DDGNN_FWD_NEPI32=$e scripts/ws_probe.cu \
    -Lpaper_2109_07893_b200 -ldgnn_b200 -Xlinker -rpath=$PWD/paper_2109_07893_b200 -o gpurun_out/probe/f32_$e &
done
wait
for kx in 64 32; do for e in 16 8; do echo -n "hp=32 epi=$e "; timeout 60 gpurun_out/probe/f32_$e $kx | tail -1; done; done
