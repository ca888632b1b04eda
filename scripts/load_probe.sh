# per-SM streaming-load probe (LDGSTS vs bulk copies against ring depth)
mkdir -p gpurun_out/probe
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 scripts/load_probe.cu -o gpurun_out/probe/load_probe && \
  timeout 300 gpurun_out/probe/load_probe
