# two-set graph mode with in-block head chaining: engine tests, 4-process parity with keep_graphs off, c2 / c5 lines
timeout 900 python -m pytest tests/test_gpu_engine.py -q -m gpu -x 2>&1 | tail -2
DGNN_KEEP_GRAPHS=0 bash scripts/mg_parity.sh 4
bash scripts/r02_cfg.sh c2 4 3
bash scripts/r02_cfg.sh c5 4 2
