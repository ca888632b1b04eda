# Build (here) K3 variants with different gather-warp counts: scripts/probe_libs/libgtc_<n>.so
set -e
mkdir -p scripts/probe_libs
OBJS=$(ls paper_2109_07893_b200/csrc/build/*.o | grep -v "/gcn_tc.o")
for g in ${G:-12 16 20 24 26}; do
  /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC \
    --expt-relaxed-constexpr -Iinclude -DDGNN_GTC_NGATHER=$g -c paper_2109_07893_b200/csrc/gcn_tc.cu -o /tmp/gtc_$g.o
  /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -o scripts/probe_libs/libgtc_$g.so $OBJS /tmp/gtc_$g.o -lcudart
done
