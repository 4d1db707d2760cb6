set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/d1_pytest.log 2>&1; tail -5 gpurun_out/d1_pytest.log
for c in ts1 sl1 wl1; do timeout 300 python tools/stamps.py $c 2>&1 | grep -v "^# wait\|^# cta"; done
