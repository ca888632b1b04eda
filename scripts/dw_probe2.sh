# weight-gradient probe: full, no MMA (1), no loads (2), no slot update (4), no split (8), combos
set -e
mkdir -p gpurun_out/probe
MASKS=${MASKS:-"0 1 2 4 8 6 5"}
for m in $MASKS; do
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -DDGNN_DW_PROBE=$m scripts/dw_probe.cu \
    -Lpaper_2109_07893_b200 -ldgnn_b200 -Xlinker -rpath=$PWD/paper_2109_07893_b200 -o gpurun_out/probe/dd$m &
done
wait
for m in $MASKS; do echo "mask $m"; timeout 60 gpurun_out/probe/dd$m 128 | tail -2; done
