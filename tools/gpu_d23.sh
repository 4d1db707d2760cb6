set -x
timeout 600 python -m pytest tests -m gpu -q -x 2>&1 | tail -2
timeout 120 python tools/bench_trace.py wl3 40
timeout 120 python tools/bench_trace.py wl2 80
timeout 300 python tools/time_run.py wl3 80 1
