set -e
mkdir -p gpurun_out/probe
V=${V:-"4:16 2:16 4:64 2:64 8:16 1:64"}
for v in $V; do gl=${v%%:*}; b=${v##*:}
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 --expt-relaxed-constexpr -DDGNN_HS_GLA=$gl -DDGNN_HS_BLK=$b \
    scripts/head_probe.cu -Lpaper_2109_07893_b200 -ldgnn_b200 -Xlinker -rpath=$PWD/paper_2109_07893_b200 -o gpurun_out/probe/hs_${gl}_$b &
done
wait
for v in $V; do gl=${v%%:*}; b=${v##*:}; timeout 60 gpurun_out/probe/hs_${gl}_$b | tail -1; done
