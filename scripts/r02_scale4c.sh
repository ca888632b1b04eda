# 4-GPU box after the early head hand-off: c2 timeline at N=4, c4 / c5 lines at N=4, c4 / c2 at N=2
timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29741 \
    bench.py --config c2 --gpus 4 --steps 2 --warmup 3 --skip-cpu --skip-e2e --timeline > gpurun_out/c2_tl4.log 2>&1; echo tl rc=$?
bash scripts/r02_cfg.sh c4 4 3
bash scripts/r02_cfg.sh c5 4 2
CUDA_VISIBLE_DEVICES=0,1 bash scripts/r02_cfg.sh c4 2 3
CUDA_VISIBLE_DEVICES=0,1 bash scripts/r02_cfg.sh c2 2 3
CUDA_VISIBLE_DEVICES=0,1 bash scripts/r02_cfg.sh c3 2 3
