for d in 0 1 2 4; do echo "== dbg=$d"; DGNN_DW_DBG=$d timeout 60 python scripts/debug_dw2.py 2>&1 | head -3; done
