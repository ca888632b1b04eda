# head_scatter sweep: lanes per active vertex (GLA) x warp threshold (HUB)
# at the configs[1] shape and a configs[2]-like heavy-tailed shape
set -e
mkdir -p gpurun_out/probe
V=${V:-"4:64 2:64 8:64 4:32 2:32 4:128"}
for c3 in 0 1; do
  for v in $V; do gl=${v%%:*}; h=${v##*:}
    nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 --expt-relaxed-constexpr -Ipaper_2109_07893_b200/csrc -Iinclude -DDGNN_HS_GLA=$gl -DDGNN_HS_HUB=$h -DHP_C3=$c3 \
      scripts/head_probe.cu -Lpaper_2109_07893_b200 -ldgnn_b200 -Xlinker -rpath=$PWD/paper_2109_07893_b200 -o gpurun_out/probe/hab_${gl}_${h}_$c3 &
  done
done
wait
for c3 in 0 1; do for v in $V; do gl=${v%%:*}; h=${v##*:}; echo -n "c3=$c3 hub=$h: "; timeout 60 gpurun_out/probe/hab_${gl}_${h}_$c3 | tail -1; done; done
