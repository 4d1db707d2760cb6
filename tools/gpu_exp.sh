for w in 8 7 6 5 4; do NUFI_EXP_IDLE=$w timeout 300 python tools/stamps.py ts1 2>&1 | head -1; done
