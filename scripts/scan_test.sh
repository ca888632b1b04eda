mkdir -p gpurun_out/probe
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -Iinclude scripts/scan_test.cu -Lpaper_2109_07893_b200 -ldgnn_b200 \
  -Xlinker -rpath=$PWD/paper_2109_07893_b200 -o gpurun_out/probe/scan_test && timeout 120 gpurun_out/probe/scan_test

