timeout 60 python scripts/debug_dw4.py; timeout 60 python scripts/debug_dw3.py 2>&1 | tail -5
for a in "64 128" "64 68" "32 36" "16 48"; do timeout 120 python scripts/debug_dw.py $a 2>&1 | grep "max rel"; done
