# per-stream busy / idle breakdown of c3 at N=4 (every rank) and N=1
mkdir -p gpurun_out
timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29741 \
    bench.py --config c3 --gpus 4 --steps 2 --warmup 3 --skip-cpu --skip-e2e --timeline > gpurun_out/c3_tl4.log 2>&1; echo n4 rc=$?
CUDA_VISIBLE_DEVICES=0 timeout 1200 python bench.py --config c3 --steps 2 --warmup 3 --skip-cpu --skip-e2e --timeline > gpurun_out/c3_tl1.log 2>&1; echo n1 rc=$?
