# d=3 shared-gather experiment: trace time on the reference's wl3 history, per build
for lib in "" pair pairF pairF1; do NUFI_LIB_VARIANT=$lib timeout 300 python tools/trace_golden.py wl3 50 5; done
