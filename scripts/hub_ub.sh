# K3 at the configs[2] shape with 8 / 16 / 32 edges per CTA slot in flight on
# rows of > 512 entries (hub_rows_kernel, DGNN_HUB_UB); libraries built here:
#   OBJS=$(ls paper_2109_07893_b200/csrc/build/*.o | grep -v /spmm.o); for u in 8 16 32; do
#     nvcc ... -DDGNN_HUB_UB=$u -c paper_2109_07893_b200/csrc/spmm.cu -o /tmp/spmm_$u.o &&
#     nvcc -shared -o scripts/probe_libs/libhub_$u.so $OBJS /tmp/spmm_$u.o -lcudart; done
for r in 1 2; do for u in 8 16 32; do
  DGNN_LIB_PATH=$PWD/scripts/probe_libs/libhub_$u.so python scripts/gcn_fwd_probe.py --c3 2>&1 | tail -1
done; done
