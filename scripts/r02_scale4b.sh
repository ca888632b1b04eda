# 4-GPU box: multi-process parity at P=4, then c2 (weak) / c4 / c5 / c3 (strong) lines at N=4, c4 at N=2
bash scripts/mg_parity.sh 4
bash scripts/r02_cfg.sh c2 4 3
bash scripts/r02_cfg.sh c4 4 3
CUDA_VISIBLE_DEVICES=0,1 bash scripts/r02_cfg.sh c4 2 3
CUDA_VISIBLE_DEVICES=0,1 bash scripts/r02_cfg.sh c2 2 3
bash scripts/r02_cfg.sh c5 4 2
bash scripts/r02_cfg.sh c3 4 3
