for d in 8 16 24; do echo "== dbg=$d"; DGNN_DW_DBG=$d timeout 60 python scripts/debug_dw4.py 2>&1 | tail -2; done
