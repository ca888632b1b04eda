# K5 at hidden 64: operand stages x landing-ring depth
set -e
mkdir -p gpurun_out/probe
V="3:6 2:8 2:10 2:12"
for v in $V; do st=${v%%:*}; rr=${v##*:}
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 --expt-relaxed-constexpr -DDGNN_FWD_ST64=$st -DDGNN_FWD_RAW64=$rr scripts/ws_probe.cu \
    -Lpaper_2109_07893_b200 -ldgnn_b200 -Xlinker -rpath=$PWD/paper_2109_07893_b200 -o gpurun_out/probe/fr_${st}_$rr &
done
wait
for kx in 128 64; do for v in $V; do st=${v%%:*}; rr=${v##*:}; echo -n "st=$st raw=$rr "; timeout 60 gpurun_out/probe/fr_${st}_$rr $kx | tail -1; done; done
