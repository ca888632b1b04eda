# head_scatter: warp-summed hub vertices (DGNN_HS_HUB=64) vs none, at the
# configs[1] shape and a (more skewed than real) configs[2] shape
set -e
mkdir -p gpurun_out/probe
for c3 in 0 1; do
  for h in 64 1000000000; do
    nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 --expt-relaxed-constexpr -Ipaper_2109_07893_b200/csrc -Iinclude -DDGNN_HS_HUB=$h -DHP_C3=$c3 \
      scripts/head_probe.cu -Lpaper_2109_07893_b200 -ldgnn_b200 -Xlinker -rpath=$PWD/paper_2109_07893_b200 -o gpurun_out/probe/hab_${h}_$c3 &
  done
done
wait
for r in 1 2; do for c3 in 0 1; do for h in 64 1000000000; do echo -n "c3=$c3 hub=$h: "; timeout 60 gpurun_out/probe/hab_${h}_$c3 | tail -1; done; done; done
