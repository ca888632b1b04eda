timeout 60 python scripts/debug_dw.py 64 128; echo rc=$?
timeout 60 python scripts/debug_dw.py 32 36; echo rc=$?
timeout 60 python scripts/debug_dw.py 16 48; echo rc=$?
