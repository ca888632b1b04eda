# early head hand-off: multi-process parity at P=4, c3 / c2 lines at N=4, c3 N=4 timeline
bash scripts/mg_parity.sh 4
bash scripts/r02_cfg.sh c3 4 3
bash scripts/r02_cfg.sh c2 4 3
timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29741 \
    bench.py --config c3 --gpus 4 --steps 2 --warmup 3 --skip-cpu --skip-e2e --timeline > gpurun_out/c3_tl4.log 2>&1; echo tl rc=$?
