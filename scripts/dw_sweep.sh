# weight-gradient kernel: L2 prefetch distance x register stages in flight (scripts/dw_probe.cu shape, kx 128)
set -e
mkdir -p gpurun_out/probe
V="0:2 128:2 256:2 512:2 1024:2 128:3 512:3"
for v in $V; do pf=${v%%:*}; pd=${v##*:}
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -DDGNN_DW_PF=$pf -DDGNN_DW_PD=$pd scripts/dw_probe.cu \
    -Lpaper_2109_07893_b200 -ldgnn_b200 -Xlinker -rpath=$PWD/paper_2109_07893_b200 -o gpurun_out/probe/dw_${pf}_$pd &
done
wait
for rep in 1 2; do for v in $V; do pf=${v%%:*}; pd=${v##*:}; echo -n "pf=$pf pd=$pd "; timeout 60 gpurun_out/probe/dw_${pf}_$pd 128 | tail -1; done; done
