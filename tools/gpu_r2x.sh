# d >= 2: 16-warp CTAs with a deeper ring (NUFI_D23_WIDE) vs the default 2 x 8-warp CTAs
for c in wl3 wl2; do
  timeout 300 python tools/trace_golden.py $c 50 5
  NUFI_D23_WIDE=1 timeout 300 python tools/trace_golden.py $c 50 5
  NUFI_D23_WIDE=1 NUFI_STAGES=3 timeout 300 python tools/trace_golden.py $c 50 5
  NUFI_D23_WIDE=1 NUFI_STAGES=2 timeout 300 python tools/trace_golden.py $c 50 5
done
NUFI_D23_WIDE=1 timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_sharded.py -m gpu -q -x -k "wl2 or wl3 or tiny or rag" 2>&1 | tail -2
