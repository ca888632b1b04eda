set -e
mkdir -p gpurun_out/probe
M=${1:-3}
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -DDGNN_DW_PROBE=$M scripts/dw_probe.cu \
    -Lpaper_2109_07893_b200 -ldgnn_b200 -Xlinker -rpath=$PWD/paper_2109_07893_b200 -o gpurun_out/probe/d$M
timeout 60 gpurun_out/probe/d$M 128
ncu --set full --clock-control none --import-source on -k regex:lstm_dw -s 1 -c 1 -o gpurun_out/dwprobe$M gpurun_out/probe/d$M 128 > gpurun_out/dwprobe_ncu.log 2>&1; echo ncu rc=$?
