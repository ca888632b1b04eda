# last refresh (4-GPU box): parity at P=4 / 2, configs[2] lines at N=4 / 2, configs[1] at N=4
bash scripts/mg_parity.sh 4
CUDA_VISIBLE_DEVICES=0,1 bash scripts/mg_parity.sh 2
bash scripts/r02_cfg.sh c3 4 3
CUDA_VISIBLE_DEVICES=0,1 bash scripts/r02_cfg.sh c3 2 3
bash scripts/r02_cfg.sh c2 4 3
