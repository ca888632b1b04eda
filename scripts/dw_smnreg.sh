# weight gradient: setmaxnreg register rebalancing x register stages in flight
set -e
mkdir -p gpurun_out/probe
V="0:2 1:2 1:3"
for v in $V; do sm=${v%%:*}; pd=${v##*:}
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -DDGNN_DW_SETMAXNREG=$sm -DDGNN_DW_PD=$pd scripts/dw_probe.cu \
    -Lpaper_2109_07893_b200 -ldgnn_b200 -Xlinker -rpath=$PWD/paper_2109_07893_b200 -o gpurun_out/probe/dsm_${sm}_$pd &
done
wait
for rep in 1 2; do for v in $V; do sm=${v%%:*}; pd=${v##*:}; echo -n "setmaxnreg=$sm pd=$pd "; timeout 20 gpurun_out/probe/dsm_${sm}_$pd 128 | tail -1; done; done
