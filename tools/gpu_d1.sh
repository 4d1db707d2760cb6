set -x
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/d1_pytest.log 2>&1; tail -3 gpurun_out/d1_pytest.log
for c in sl1 ts1 wl1; do timeout 300 python tools/stamps.py $c 2>&1 | grep -v "^  n=\|TMA wait"; done
