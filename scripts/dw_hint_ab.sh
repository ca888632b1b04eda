# A/B: weight-gradient kernel with and without the L2 eviction hints, interleaved runs
set -e
mkdir -p gpurun_out/probe
for h in 0 1; do
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -DDGNN_DW_HINTS=$h scripts/dw_probe.cu \
    -Lpaper_2109_07893_b200 -ldgnn_b200 -Xlinker -rpath=$PWD/paper_2109_07893_b200 -o gpurun_out/probe/dh$h &
done
wait
for rep in 1 2 3; do for h in 0 1; do echo -n "hints=$h "; timeout 60 gpurun_out/probe/dh$h 128 | tail -1; done; done
