import ctypes, os, sys, time
sys.path.insert(0, "/root/repo")
import torch
import paper_2301_05581_b200 as nufi
from paper_2301_05581_b200 import _lib
from paper_2301_05581_b200.configs import workload
from paper_2301_05581_b200.spline import _placeholder_ic
w = workload("wl1")
lib = _lib.load()
for it in range(7):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    cfg = _lib.make_config(w.grid, _placeholder_ic(w.grid), w.tau, w.n_steps, rho_bar=1.0)
    t1 = time.perf_counter()
    h = ctypes.c_void_p()
    lib.nufi_create(ctypes.byref(cfg), 0, None, ctypes.byref(h))
    t2 = time.perf_counter()
    lib.nufi_sync(h)
    t3 = time.perf_counter()
    cfg2 = _lib.make_config(w.grid, w.ic, w.tau, w.n_steps, rho_bar=None)
    lib.nufi_set_initial_condition(h, ctypes.byref(cfg2))
    t4 = time.perf_counter()
    lib.nufi_destroy(h)
    t5 = time.perf_counter()
    if it >= 2:
        print(f"cfg {1e6*(t1-t0):.0f} us  nufi_create {1e6*(t2-t1):.0f} us  sync {1e6*(t3-t2):.0f} us  set_ic {1e6*(t4-t3):.0f} us  destroy {1e6*(t5-t4):.0f} us", flush=True)
# the same with a caller stream (no stream create / destroy inside the library)
s = torch.cuda.Stream()
for it in range(7):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    cfg = _lib.make_config(w.grid, _placeholder_ic(w.grid), w.tau, w.n_steps, rho_bar=1.0)
    t1 = time.perf_counter()
    h = ctypes.c_void_p()
    lib.nufi_create(ctypes.byref(cfg), 0, ctypes.c_void_p(s.cuda_stream), ctypes.byref(h))
    t2 = time.perf_counter()
    lib.nufi_sync(h)
    t3 = time.perf_counter()
    lib.nufi_destroy(h)
    t5 = time.perf_counter()
    if it >= 2:
        print(f"caller stream: nufi_create {1e6*(t2-t1):.0f} us  sync {1e6*(t3-t2):.0f} us  destroy {1e6*(t5-t3):.0f} us", flush=True)
