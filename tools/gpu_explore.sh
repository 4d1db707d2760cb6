set -x
mkdir -p gpurun_out
for c in ts1 sl1 wl1; do timeout 300 python tools/stamps.py $c; done > gpurun_out/e_stamps.log 2>&1
( timeout 120 python tools/bench_trace.py wl3 40
  NUFI_PASSES=2 timeout 120 python tools/bench_trace.py wl3 40
  NUFI_PASSES=8 timeout 120 python tools/bench_trace.py wl3 40
  NUFI_PPT=1 NUFI_PASSES=8 timeout 120 python tools/bench_trace.py wl3 40
  NUFI_SPS=2 NUFI_STAGES=2 timeout 120 python tools/bench_trace.py wl3 40
  timeout 120 python tools/bench_trace.py wl2 80
  NUFI_PPT=1 timeout 120 python tools/bench_trace.py wl2 80
  NUFI_SPS=2 timeout 120 python tools/bench_trace.py wl2 80
  NUFI_SPS=8 NUFI_STAGES=3 timeout 120 python tools/bench_trace.py wl2 80
) > gpurun_out/e_trace.log 2>&1
cat gpurun_out/e_stamps.log | grep -v "^#" | head -40
cat gpurun_out/e_trace.log
