for ps in 1 2 4; do NUFI_PASSES=$ps timeout 120 python tools/bench_trace.py wl2 80; done
for ps in 2 4 8; do NUFI_PASSES=$ps timeout 120 python tools/bench_trace.py wl3 40; done
NUFI_SPS=2 timeout 120 python tools/bench_trace.py wl3 40
NUFI_STAGES=3 NUFI_SPS=2 timeout 120 python tools/bench_trace.py wl3 40
