# c3 (tm-gcn, strong scaling) at N=4 and N=2 with the current kernels
bash scripts/r02_cfg.sh c3 4 3
CUDA_VISIBLE_DEVICES=0,1 bash scripts/r02_cfg.sh c3 2 3
