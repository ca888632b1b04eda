# TMEM-operand weight-gradient probe: full, no MMA (1), no HBM reads (2), no slot update (4), no TMEM stores (8)
set -e
mkdir -p gpurun_out/probe
MASKS=${MASKS:-"0 1 2 4 8 3 11"}
for m in $MASKS; do
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -DDGNN_DTS_PROBE=$m scripts/dts_probe.cu \
    -Lpaper_2109_07893_b200 -ldgnn_b200 -Xlinker -rpath=$PWD/paper_2109_07893_b200 -o gpurun_out/probe/ts$m &
done
wait
for kx in 128 68; do for m in $MASKS; do timeout 60 gpurun_out/probe/ts$m $kx | tail -1; done; done
