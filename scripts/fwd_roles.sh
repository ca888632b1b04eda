# forward LSTM kernel (K5) at configs[1] shapes: producer / epilogue warp counts
set -e
mkdir -p gpurun_out/probe
V=${V:-"8:16 16:8 8:8 4:16"}
for v in $V; do p=${v%%:*}; e=${v##*:}
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 --expt-relaxed-constexpr -DDGNN_FWD_NPROD=$p -DDGNN_FWD_NEPI64=$e scripts/ws_probe.cu \
    -Lpaper_2109_07893_b200 -ldgnn_b200 -Xlinker -rpath=$PWD/paper_2109_07893_b200 -o gpurun_out/probe/f_${p}_$e &
done
wait
for kx in 128 64; do for v in $V; do p=${v%%:*}; e=${v##*:}; echo -n "prod=$p epi=$e "; timeout 60 gpurun_out/probe/f_${p}_$e $kx | tail -1; done; done
