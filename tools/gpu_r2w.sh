# A/B: current build vs libnufi_b200_old.so (HEAD) on the d>=2 traces + wl2/wl3 bench
for lib in old "" old ""; do
  NUFI_LIB_VARIANT=$lib timeout 300 python tools/trace_golden.py wl3 50 5
  NUFI_LIB_VARIANT=$lib timeout 300 python tools/trace_golden.py wl2 50 5
done
timeout 900 python -m pytest tests/test_gpu_api_surface.py tests/test_gpu_parity.py -m gpu -q -x 2>&1 | tail -2
