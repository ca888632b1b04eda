# 4-GPU box: c4 at N=4 and 2, c5 at N=4, c2 at N=4 (weak)
bash scripts/r02_cfg.sh c4 4 2
CUDA_VISIBLE_DEVICES=0,1 bash scripts/r02_cfg.sh c4 2 2
bash scripts/r02_cfg.sh c5 4 2
bash scripts/r02_cfg.sh c2 4 3
