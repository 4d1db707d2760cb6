set -x
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/d23_pytest.log 2>&1; tail -3 gpurun_out/d23_pytest.log
timeout 120 python tools/bench_trace.py wl3 40
timeout 120 python tools/bench_trace.py wl2 80
timeout 120 python tools/bench_trace.py wl2 150
