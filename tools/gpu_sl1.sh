set -x
timeout 600 python -m pytest tests -m gpu -q -x 2>&1 | tail -2
timeout 300 python tools/stamps.py ts1 2>&1 | grep -v "^  n="
timeout 300 python tools/stamps.py sl1 2>&1 | grep -v "^  n="
NUFI_D1_SPS=2 NUFI_D1_STAGES=4 timeout 300 python tools/stamps.py sl1 2>&1 | grep -v "^  n="
NUFI_D1_SPS=1 NUFI_D1_STAGES=8 timeout 300 python tools/stamps.py sl1 2>&1 | grep -v "^  n="
NUFI_D1_SPS=2 NUFI_D1_STAGES=3 timeout 300 python tools/stamps.py sl1 2>&1 | grep -v "^  n="
