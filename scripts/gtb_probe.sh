# Build (here) the BWD rows-kernel probe libraries: scripts/probe_libs/libgtb_<mask>.so
set -e
mkdir -p scripts/probe_libs
OBJS=$(ls paper_2109_07893_b200/csrc/build/*.o | grep -v gcn_tc.o)
for m in ${MASKS:-1 2 4 8 5}; do
  /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC \
    --expt-relaxed-constexpr -Iinclude -DDGNN_GTB_PROBE=$m -c paper_2109_07893_b200/csrc/gcn_tc.cu -o /tmp/gtb_$m.o
  /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -o scripts/probe_libs/libgtb_$m.so $OBJS /tmp/gtb_$m.o -lcudart
done
