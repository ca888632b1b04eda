set -e
mkdir -p gpurun_out/probe
for m in 16 18; do
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -DDGNN_DW_PROBE=$m scripts/dw_probe.cu \
    -Lpaper_2109_07893_b200 -ldgnn_b200 -Xlinker -rpath=$PWD/paper_2109_07893_b200 -o gpurun_out/probe/d$m
done
for m in 16 18; do timeout 60 gpurun_out/probe/d$m 128; done

