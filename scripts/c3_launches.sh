# c3 N=1: uninstrumented launch list (ncu, serialized) of one timed epoch + timeline
mkdir -p gpurun_out
KERNELS="" bash scripts/profile_r02.sh c3
timeout 1200 python bench.py --config c3 --steps 2 --warmup 3 --skip-cpu --skip-e2e --timeline > gpurun_out/c3_tl1.log 2>&1; echo tl rc=$?
