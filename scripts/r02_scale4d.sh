# 4-GPU box, latest kernels: multi-process parity at P=4 / P=2, then every config line at N=4 / N=2
bash scripts/mg_parity.sh 4
CUDA_VISIBLE_DEVICES=0,1 bash scripts/mg_parity.sh 2
for c in c2 c3 c4; do bash scripts/r02_cfg.sh $c 4 3; CUDA_VISIBLE_DEVICES=0,1 bash scripts/r02_cfg.sh $c 2 3; done
bash scripts/r02_cfg.sh c5 4 2
