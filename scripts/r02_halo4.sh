# 4-GPU box: multi-process parity with the tm-gcn halo at P=4 and P=2, then c3 lines at N=4 / N=2
bash scripts/mg_parity.sh 4
CUDA_VISIBLE_DEVICES=0,1 bash scripts/mg_parity.sh 2
bash scripts/r02_cfg.sh c3 4 3
CUDA_VISIBLE_DEVICES=0,1 bash scripts/r02_cfg.sh c3 2 3
