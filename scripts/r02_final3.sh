# refresh after the narrow-operand kernel changes: c3 / c4 at N=1, then (4-GPU box) parity + N=2/4 lines
bash scripts/r02_cfg.sh c3 1 3
bash scripts/r02_cfg.sh c4 1 2
bash scripts/mg_parity.sh 4
for c in c3 c4; do bash scripts/r02_cfg.sh $c 4 3; CUDA_VISIBLE_DEVICES=0,1 bash scripts/r02_cfg.sh $c 2 3; done
bash scripts/r02_cfg.sh c5 4 2
