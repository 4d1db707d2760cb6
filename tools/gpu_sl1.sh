set -x
timeout 600 python -m pytest tests -m gpu -q -x 2>&1 | tail -2
timeout 300 python tools/stamps.py ts1 2>&1 | grep -v "^  n=\|tail phases"
for st in 2 3 4; do NUFI_D1_STAGES=$st timeout 300 python tools/stamps.py sl1 2>&1 | grep -v "^  n=\|tail phases"; done
NUFI_D1_STAGES=6 timeout 300 python tools/stamps.py ts1 2>&1 | grep -v "^  n=\|tail phases"
