for d in 0 1; do echo "== dbg=$d"; DGNN_DW_DBG=$d timeout 60 python scripts/debug_dw3.py 2>&1 | tail -6; done
DGNN_DW_DBG=2 timeout 60 python scripts/debug_dw2.py 2>&1 | tail -3
