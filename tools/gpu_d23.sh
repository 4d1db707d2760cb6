set -x
timeout 600 python -m pytest tests -m gpu -q -x 2>&1 | tail -2
timeout 120 python tools/bench_trace.py wl3 40
NUFI_WARPS=16 timeout 120 python tools/bench_trace.py wl3 40
NUFI_WARPS=16 NUFI_STAGES=3 timeout 120 python tools/bench_trace.py wl3 40
NUFI_WARPS=16 NUFI_PASSES=2 timeout 120 python tools/bench_trace.py wl3 40
timeout 120 python tools/bench_trace.py wl2 80
NUFI_WARPS=16 timeout 120 python tools/bench_trace.py wl2 80
NUFI_WARPS=16 NUFI_STAGES=3 timeout 120 python tools/bench_trace.py wl2 80
