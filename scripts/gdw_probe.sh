# GCN weight gradient: loader x converter warp counts
set -e
mkdir -p gpurun_out/probe
V=${V:-"8:4 8:8 4:4 4:8 8:12"}
for v in $V; do l=${v%%:*}; c=${v##*:}
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -Iinclude -DDGNN_GDW_NLOAD=$l -DDGNN_GDW_NCONV=$c \
    scripts/gdw_probe.cu -Lpaper_2109_07893_b200 -ldgnn_b200 -Xlinker -rpath=$PWD/paper_2109_07893_b200 -o gpurun_out/probe/gdw_${l}_$c &
done
wait
for rep in 1 2; do for v in $V; do l=${v%%:*}; c=${v##*:}; timeout 60 gpurun_out/probe/gdw_${l}_$c | tail -1; done; done
