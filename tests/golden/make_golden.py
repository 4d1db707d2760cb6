"""Generate golden fixtures by running the UNMODIFIED reference (vpflow) in this container.

Test infrastructure only. This script imports the reference package from
/root/reference/pkg/src (read-only) and records, per BASELINE config, the
outputs of the canonical per-step loop (reference has no
driver, the loop follows SPEC.md:465-468):

    r = density.compute_rho(ctx, n)                  # density.py:72-91
    phi, spec = poisson.solve_poisson(r.density)     # poisson.py:90-112
    fit = spline.fit_spline(phi, grid)               # spline.py:71-86
    hist.append(fit)                                 # spline.py:132-142
    W = poisson.electric_energy(spec)                # poisson.py:115-120
    E = kernels.eval_E_many(fit.coeffs, L, x_node_matrix(grid))   # kernels.py:102-123

It also records trace goldens: seeded random (x, v) pushed through a real
history by kernels.trace_backward (kernels.py:390-412, numba backend) with
half_kick 0 and 1.

The fixtures are committed under tests/golden/*.npz; the GPU box never runs
this script (/root/reference does not exist there).

Usage:  python tests/golden/make_golden.py wl1 ts1 ...   (default: all)
"""

from __future__ import annotations

import json
import math
import os
import platform
import sys
import time

import numpy as np

REF = "/root/reference/pkg/src"
OUT = os.path.dirname(os.path.abspath(__file__))

# Config table: SURVEY.md §8(d) / BASELINE.json configs. "keep" = number of
# steps (0..keep-1) whose rho/coeffs/E are stored; W and stats are stored for
# every step that was run.
CONFIGS = {
    # BASELINE configs
    "wl1": dict(d=1, Nx=64, Nv=256, vmax=6.0, tau=1 / 8, N=240, bench="weak_landau_1d", alpha=None, keep=51),
    "ts1": dict(d=1, Nx=64, Nv=512, vmax=10.0, tau=1 / 16, N=1600, bench="two_stream_1d", alpha=None, keep=51),
    "sl1": dict(d=1, Nx=256, Nv=2048, vmax=8.0, tau=1 / 16, N=800, bench="weak_landau_1d", alpha=0.5, keep=51),
    "wl2": dict(d=2, Nx=32, Nv=64, vmax=6.0, tau=1 / 8, N=160, bench="strong_landau_2d", alpha=0.01, keep=51),
    # full size to t_end (80 steps, ~3 h of numba on 8 cores); the fixture is rewritten
    # every few steps, truncated to the steps done, so a cut-off run still pins 0..n
    "wl3": dict(d=3, Nx=16, Nv=32, vmax=6.0, tau=1 / 8, N=80, bench="weak_landau_3d", alpha=0.01, keep=51,
                save_every=2),
    # reduced / small cases (fast parity cases; oracle finishes in seconds)
    "wl3r": dict(d=3, Nx=16, Nv=8, vmax=6.0, tau=1 / 8, N=80, bench="weak_landau_3d", alpha=0.01, keep=81),
    "kat_wl": dict(d=1, Nx=32, Nv=128, vmax=10.0, tau=1 / 16, N=160, bench="weak_landau_1d", alpha=None, keep=161),
    "tiny2": dict(d=2, Nx=8, Nv=8, vmax=6.0, tau=1 / 8, N=24, bench="strong_landau_2d", alpha=0.5, keep=25),
    "tiny3": dict(d=3, Nx=8, Nv=4, vmax=6.0, tau=1 / 8, N=12, bench="two_stream_3d", alpha=None, keep=13),
    "eq1": dict(d=1, Nx=32, Nv=128, vmax=10.0, tau=1 / 16, N=160, bench="weak_landau_1d", alpha=0.0, keep=1),
    # ragged / non-power-of-two grids (generic-N kernel paths, Nv^d not a multiple of 32 or 8)
    "rag1": dict(d=1, Nx=24, Nv=40, vmax=6.0, tau=1 / 8, N=40, bench="weak_landau_1d", alpha=0.05, keep=41),
    "rag2": dict(d=2, Nx=6, Nv=10, vmax=6.0, tau=1 / 8, N=16, bench="strong_landau_2d", alpha=0.3, keep=17),
    "rag3": dict(d=3, Nx=5, Nv=3, vmax=5.0, tau=1 / 8, N=8, bench="weak_landau_3d", alpha=0.05, keep=9),
    # grids beyond one CTA (Nx^d > 4096: multi-CTA tail; slabs > 100 KB: in-place trace)
    "big1": dict(d=1, Nx=5000, Nv=16, vmax=6.0, tau=1 / 8, N=6, bench="weak_landau_1d", alpha=0.05, keep=7),
    "big2": dict(d=2, Nx=72, Nv=6, vmax=6.0, tau=1 / 8, N=6, bench="strong_landau_2d", alpha=0.2, keep=7),
    "big2g": dict(d=2, Nx=120, Nv=4, vmax=6.0, tau=1 / 8, N=4, bench="strong_landau_2d", alpha=0.2, keep=5),
    "big3": dict(d=3, Nx=22, Nv=3, vmax=5.0, tau=1 / 8, N=4, bench="weak_landau_3d", alpha=0.05, keep=5),
    # FP32 history mode (PotentialHistory(dtype=float32), spline.py:118-125)
    "kat_wl_f32": dict(d=1, Nx=32, Nv=128, vmax=10.0, tau=1 / 16, N=160, bench="weak_landau_1d", alpha=None,
                       keep=161, dtype="float32"),
    "tiny2_f32": dict(d=2, Nx=8, Nv=8, vmax=6.0, tau=1 / 8, N=24, bench="strong_landau_2d", alpha=0.5, keep=25,
                      dtype="float32"),
}


# history length used for the trace goldens
TRACE_N = {"kat_wl": 40, "tiny2": 20, "tiny3": 12, "wl3r": 16, "rag1": 30, "rag2": 12, "rag3": 7, "big3": 3}


def build(cfg):
    from vpflow.grids import GridSpec
    from vpflow.initial import InitialCondition, VelocityProfile, make_benchmark

    d = cfg["d"]
    if cfg["bench"] == "two_stream_3d":
        # 3-d two-stream needs L = 10*pi (initial.py:115); smaller grid here
        L = 10.0 * math.pi
        ic = make_benchmark("two_stream_3d")
    else:
        L = 4.0 * math.pi
        if cfg["bench"] == "weak_landau_3d":
            # not a reference built-in; SURVEY.md §0 fact 10 / §8(d)
            ic = InitialCondition(benchmark="weak_landau_3d", d=3, L=L, alpha=cfg["alpha"], k=0.5,
                                  profiles=(VelocityProfile(),) * 3)
        elif cfg["alpha"] is not None:
            ic = make_benchmark(cfg["bench"], alpha=cfg["alpha"])
        else:
            ic = make_benchmark(cfg["bench"])
    g = GridSpec(d=d, L=L, Nx=cfg["Nx"], Nv=cfg["Nv"], vmax=cfg["vmax"])
    return g, ic


def ic_descriptor(ic):
    return dict(benchmark=ic.benchmark, d=ic.d, L=ic.L, alpha=ic.alpha, k=ic.k,
                profiles=[dict(centers=list(p.centers), weights=list(p.weights), power=p.power)
                          for p in ic.profiles])


def run(name, cfg):
    from vpflow import density, kernels, poisson, spline
    from vpflow.flow import FlowContext
    from vpflow.grids import x_node_matrix

    g, ic = build(cfg)
    tau = cfg["tau"]
    N = cfg["N"]
    keep = cfg["keep"]
    hist = spline.PotentialHistory(g, tau, dtype=np.dtype(cfg.get("dtype", "float64")))
    ctx = FlowContext(history=hist, ic=ic, tau=tau, grid=g)
    Xn = x_node_matrix(g)
    nodes = g.n_nodes
    rho = np.zeros((keep, nodes))
    coeffs = np.zeros((keep, nodes))
    E = np.zeros((keep, nodes, g.d))
    W = np.zeros(N + 1)
    stats = np.zeros((N + 1, 3))
    t_rho = np.zeros(N + 1)
    t_tail = np.zeros(N + 1)
    evals = []
    t0 = time.time()
    for n in range(N + 1):
        a = time.perf_counter()
        r = density.compute_rho(ctx, n)
        b = time.perf_counter()
        phi, spec = poisson.solve_poisson(r.density)
        fit = spline.fit_spline(phi, g)
        hist.append(fit)
        W[n] = poisson.electric_energy(spec)
        c = time.perf_counter()
        t_rho[n] = b - a
        t_tail[n] = c - b
        stats[n] = (r.neutralization, r.f_min, r.f_max)
        evals.append(ctx.field_evals)
        if n < keep:
            rho[n] = r.density.values.reshape(-1)
            coeffs[n] = np.asarray(hist.entry(n).coeffs, dtype=np.float64).reshape(-1)  # the stored slab
            E[n] = kernels.eval_E_many(fit.coeffs, g.L, Xn)
        if cfg.get("save_every") and n % cfg["save_every"] == 0 and n < N:
            save(name, cfg, g, ic, ctx, n, keep, rho, coeffs, E, W, stats, t_rho, t_tail, evals, t0)
        if n % 50 == 0 or cfg.get("save_every"):
            print(f"[{name}] step {n}/{N}  W={W[n]:.6e}  t={time.time() - t0:.1f}s", flush=True)
    save(name, cfg, g, ic, ctx, N, keep, rho, coeffs, E, W, stats, t_rho, t_tail, evals, t0)
    print(f"[{name}] done in {time.time() - t0:.1f}s", flush=True)
    return g, ic, hist


def save(name, cfg, g, ic, ctx, n, keep, rho, coeffs, E, W, stats, t_rho, t_tail, evals, t0):
    """Write the fixture for steps 0..n (W/stats for every step run, rho/coeffs/E for min(keep, n+1))."""
    k = min(keep, n + 1)
    np.savez_compressed(
        os.path.join(OUT, f"{name}.npz"),
        rho=rho[:k], coeffs=coeffs[:k], E=E[:k], W=W[: n + 1], stats=stats[: n + 1], t_rho=t_rho[: n + 1],
        t_tail=t_tail[: n + 1], field_evals=np.array(evals[: n + 1], dtype=np.int64), rho_bar=np.array(ctx.rho_bar),
    )
    meta = dict(name=name, cfg=cfg, steps_done=n, L=g.L, ic=ic_descriptor(ic), rho_bar=ctx.rho_bar,
                wall_s=time.time() - t0, rho_s=float(t_rho[: n + 1].sum()), tail_s=float(t_tail[: n + 1].sum()),
                field_evals=int(evals[n]), host=host_info())
    with open(os.path.join(OUT, f"{name}.json"), "w") as fh:
        json.dump(meta, fh, indent=1)


def trace_goldens(name, g, stack, tau, n, M=2000, seed=1234):
    """Seeded points through a stored history (stack: (rows, Nx, ..)) with both half_kick values."""
    from vpflow import kernels

    rng = np.random.default_rng(seed)
    d = g.d
    X0 = rng.uniform(0.0, g.L, size=(M, d))
    V0 = rng.uniform(-g.vmax, g.vmax, size=(M, d))
    stack = np.ascontiguousarray(stack)
    out = {"Xin": X0, "Vin": V0, "coeffs": stack[: n + 1].reshape(n + 1, -1), "n": np.array(n)}
    for hk in (0, 1):
        X = X0.copy()
        V = V0.copy()
        ev = kernels.trace_backward(stack[: n + 1] if hk else stack[:n], g.L, n, tau, X, V, bool(hk))
        out[f"X{hk}"] = X
        out[f"V{hk}"] = V
        out[f"evals{hk}"] = np.array(ev)
    # numpy twin on the same inputs (reference's in-tree second backend)
    kernels.set_backend("numpy")
    for hk in (0, 1):
        X = X0.copy()
        V = V0.copy()
        kernels.trace_backward(stack[: n + 1] if hk else stack[:n], g.L, n, tau, X, V, bool(hk))
        out[f"Xnp{hk}"] = X
        out[f"Vnp{hk}"] = V
    kernels.set_backend("numba")
    np.savez_compressed(os.path.join(OUT, f"trace_{name}.npz"), L=np.array(g.L), tau=np.array(tau), **out)


# steps at which the observable sweep goldens are taken (Psi needs fields 0..n)
SWEEP_N = {"kat_wl": (0, 1, 20, 40), "tiny2": (0, 3, 10, 20), "tiny3": (0, 2, 6, 11), "wl3r": (0, 5, 16),
           "rag1": (0, 7, 30), "rag2": (0, 5, 15), "rag3": (0, 3, 7)}


def conserved_weights():
    """The conserved-quantity weights of SPEC.md:403-406 as quadrature_sweep weights
    (f, f^2, f ln f with 0 ln 0 := 0, |v|^2 f / 2, v f)."""

    def f_ln_f(X, V, F):
        safe = np.where(F > 0, F, 1.0)
        return np.where(F > 0, F * np.log(safe), 0.0)

    return [
        lambda X, V, F: F,
        lambda X, V, F: F * F,
        f_ln_f,
        lambda X, V, F: 0.5 * np.sum(V * V, axis=1) * F,
        lambda X, V, F: V * F[:, None],
    ]


def sweep_goldens(name, g, ic, stack, tau):
    """density.quadrature_sweep_many (density.py:104-120, numba backend) with the
    conserved-quantity weights at the steps SWEEP_N[name], through a stored history."""
    from vpflow import density, spline
    from vpflow.flow import FlowContext

    hist = spline.PotentialHistory(g, tau)
    for c in stack:
        hist.append(spline.SplineField(grid=g, coeffs=np.ascontiguousarray(c)))
    ctx = FlowContext(history=hist, ic=ic, tau=tau, grid=g)
    steps = [n for n in SWEEP_N[name] if n + 1 <= len(stack)]
    rows = []
    evals = []
    for n in steps:
        ctx.field_evals = 0
        f, f2, flnf, kin, mom = density.quadrature_sweep_many(ctx, n, conserved_weights())
        rows.append([f, f2, flnf, kin] + list(np.atleast_1d(mom)))
        evals.append(ctx.field_evals)
    np.savez_compressed(os.path.join(OUT, f"sweep_{name}.npz"), steps=np.array(steps), moments=np.array(rows),
                        field_evals=np.array(evals, dtype=np.int64),
                        columns=np.array(["f", "f2", "f_ln_f", "kinetic"] + [f"mom{a}" for a in range(g.d)]))


def checkpoint_goldens():
    """VPHIST01 files written by the reference's PotentialHistory.save (spline.py:157-169)."""
    from vpflow import spline

    for base, rows, dtype in (("kat_wl", 20, "float64"), ("tiny2_f32", 10, "float32")):
        g, _ = build(CONFIGS[base])
        z = np.load(os.path.join(OUT, f"{base}.npz"))
        stack = z["coeffs"].reshape((-1,) + (g.Nx,) * g.d)[:rows]
        hist = spline.PotentialHistory(g, CONFIGS[base]["tau"], dtype=np.dtype(dtype))
        for c in stack:
            hist.append(spline.SplineField(grid=g, coeffs=np.ascontiguousarray(c)))
        hist.save(os.path.join(OUT, f"{base}_{rows}.vphist"))


FIELD_SLOT = {"kat_wl": 20, "tiny2": 10, "tiny3": 6, "rag1": 12, "rag2": 8, "rag3": 5}


def field_goldens():
    """SplineField.eval_phi_many / eval_E_many (spline.py:46-52 -> kernels.py:84-123) of one
    stored slab at seeded points plus edge positions (0, L, -tiny, nodes, far images)."""
    from vpflow import spline

    for base, slot in FIELD_SLOT.items():
        g, _ = build(CONFIGS[base])
        z = np.load(os.path.join(OUT, f"{base}.npz"))
        c = z["coeffs"][slot].reshape((g.Nx,) * g.d)
        fld = spline.SplineField(grid=g, coeffs=c)
        rng = np.random.default_rng(99)
        X = rng.uniform(-3 * g.L, 4 * g.L, size=(600, g.d))
        edge = np.array([0.0, g.L, -1e-300, -5e-17, g.L * (1 - 1e-16), g.L / g.Nx, 3 * g.L / g.Nx, -g.L, 7 * g.L])
        E = np.stack([np.resize(edge, 60)] * g.d, axis=1)
        for a in range(g.d):
            E[:, a] = np.roll(E[:, a], a)
        X = np.concatenate([X, E])
        np.savez_compressed(os.path.join(OUT, f"field_{base}.npz"), X=X, slot=np.array(slot),
                            phi=fld.eval_phi_many(X), E=fld.eval_E_many(X))


HOOK_CASES = {"kat_wl": (12, (3, 7)), "tiny2": (8, (2, 5)), "tiny3": (6, (1, 4))}


def hook_goldens():
    """FlowContext.install_field(step, UniformField(E0)) (flow.py:44-47, spline.py:55-68):
    the reference's generic trace (flow.py:65-82) through a stored history with two slots
    overridden, psi_batch and psi_tilde_batch at seeded points; plus the all-uniform
    constant-force case."""
    from vpflow import flow, spline

    for base, (n, slots) in HOOK_CASES.items():
        g, ic = build(CONFIGS[base])
        tau = CONFIGS[base]["tau"]
        z = np.load(os.path.join(OUT, f"{base}.npz"))
        stack = z["coeffs"].reshape((-1,) + (g.Nx,) * g.d)[: n + 1]
        hist = spline.PotentialHistory(g, tau)
        for c in stack:
            hist.append(spline.SplineField(grid=g, coeffs=np.ascontiguousarray(c)))
        ctx = flow.FlowContext(history=hist, ic=ic, tau=tau, grid=g)
        rng = np.random.default_rng(2024)
        E0 = rng.uniform(-0.4, 0.4, (len(slots), g.d))
        for s_, e in zip(slots, E0):
            ctx.install_field(s_, spline.UniformField(e))
        x = rng.uniform(-g.L, 2 * g.L, (400, g.d))
        v = rng.uniform(-g.vmax, g.vmax, (400, g.d))
        X1, V1 = flow.psi_batch(ctx, n, x, v)
        X0, V0 = flow.psi_tilde_batch(ctx, n, x, v)
        # all slots uniform: the constant-force closed form
        ctx_u = flow.FlowContext(history=spline.PotentialHistory(g, tau), ic=ic, tau=tau, grid=g)
        Eu = rng.uniform(-0.4, 0.4, g.d)
        for k in range(n + 1):
            ctx_u.install_field(k, spline.UniformField(Eu))
        XU, VU = flow.psi_batch(ctx_u, n, x, v)
        np.savez_compressed(os.path.join(OUT, f"hook_{base}.npz"), n=np.array(n), slots=np.array(slots), E0=E0,
                            x=x, v=v, X_psi=X1, V_psi=V1, X_tilde=X0, V_tilde=V0, E_uniform=Eu, X_uniform=XU,
                            V_uniform=VU, evals=np.array(ctx.field_evals))


API_ICS = ("weak_landau_1d", "two_stream_1d", "strong_landau_2d", "two_stream_3d", "weak_landau_3d")


def api_goldens():
    """The reference's module-level API beyond the loop (the drop-in surface a vpflow caller
    imports): initial.eval_f0 / background_density (initial.py:165-208), kernels.bspline_weights
    / bspline_dweights (kernels.py:62-81), poisson.transform_values / inverse_transform
    (poisson.py:72-87) on seeded inputs."""
    from vpflow import initial, kernels, poisson
    from vpflow.grids import GridSpec
    from vpflow.initial import InitialCondition, VelocityProfile, make_benchmark

    rng = np.random.default_rng(314)
    out = {}
    for name in API_ICS:
        if name == "weak_landau_3d":
            ic = InitialCondition(benchmark=name, d=3, L=4 * math.pi, alpha=0.01, k=0.5,
                                  profiles=(VelocityProfile(),) * 3)
        else:
            ic = make_benchmark(name)
        d = ic.d
        x = rng.uniform(-2 * ic.L, 3 * ic.L, (700, d))
        v = rng.uniform(-9.0, 9.0, (700, d))
        out[f"f0_{name}_x"] = x
        out[f"f0_{name}_v"] = v
        out[f"f0_{name}_F"] = initial.eval_f0(ic, x, v)
        xb = rng.uniform(0, ic.L, (3, 5, d))
        vb = rng.normal(0, 2, (3, 5, d))
        out[f"f0b_{name}_x"] = xb
        out[f"f0b_{name}_v"] = vb
        out[f"f0b_{name}_F"] = initial.eval_f0(ic, xb, vb)
    for cname in ("wl1", "ts1", "sl1", "wl2", "wl3", "wl3r", "tiny3", "rag2"):
        g, ic = build(CONFIGS[cname])
        out[f"rhobar_{cname}"] = np.array(initial.background_density(ic, g))
    t = np.concatenate([rng.uniform(0, 1, 997), [0.0, 1.0, 1e-300, 1 - 1e-16, 0.5, 0.25]])
    out["bs_t"] = t
    out["bs_w"] = kernels.bspline_weights(t)
    out["bs_dw"] = kernels.bspline_dweights(t)
    t2 = rng.uniform(0, 1, (7, 9))
    out["bs_t2"] = t2
    out["bs_w2"] = kernels.bspline_weights(t2)
    out["bs_dw2"] = kernels.bspline_dweights(t2)
    for d, N in ((1, 32), (1, 5), (2, 8), (2, 6), (3, 8), (3, 5)):
        g = GridSpec(d=d, L=4 * math.pi, Nx=N, Nv=4, vmax=6.0)
        vals = rng.normal(0, 1, g.shape_x)
        spec = poisson.transform_values(g, vals)
        out[f"tr_{d}_{N}_in"] = vals
        out[f"tr_{d}_{N}_spec"] = spec.coeffs
        cplx = rng.normal(0, 1, g.shape_x) + 1j * rng.normal(0, 1, g.shape_x)
        out[f"tr_{d}_{N}_cin"] = cplx
        out[f"tr_{d}_{N}_inv"] = poisson.inverse_transform(poisson.SpectralField(grid=g, coeffs=cplx))
    np.savez_compressed(os.path.join(OUT, "api.npz"), **out)


def hook_spline_goldens():
    """FlowContext.install_field(step, SplineField) (flow.py:44-47): stored slots replaced by
    OTHER steps' spline fields (plus one UniformField), then psi_batch / psi_tilde_batch
    through the reference's generic trace (flow.py:65-82)."""
    from vpflow import flow, spline

    for base, (n, slots) in HOOK_CASES.items():
        g, ic = build(CONFIGS[base])
        tau = CONFIGS[base]["tau"]
        z = np.load(os.path.join(OUT, f"{base}.npz"))
        stack = z["coeffs"].reshape((-1,) + (g.Nx,) * g.d)
        hist = spline.PotentialHistory(g, tau)
        for c in stack[: n + 1]:
            hist.append(spline.SplineField(grid=g, coeffs=np.ascontiguousarray(c)))
        ctx = flow.FlowContext(history=hist, ic=ic, tau=tau, grid=g)
        rng = np.random.default_rng(2025)
        src = [int(s) + n // 2 + 1 for s in slots]  # a later step's field in each slot
        for s_, k in zip(slots, src):
            ctx.install_field(s_, spline.SplineField(grid=g, coeffs=np.ascontiguousarray(stack[k])))
        Eu = rng.uniform(-0.3, 0.3, g.d)
        ctx.install_field(n - 1, spline.UniformField(Eu))
        x = rng.uniform(-g.L, 2 * g.L, (300, g.d))
        v = rng.uniform(-g.vmax, g.vmax, (300, g.d))
        X1, V1 = flow.psi_batch(ctx, n, x, v)
        X0, V0 = flow.psi_tilde_batch(ctx, n, x, v)
        np.savez_compressed(os.path.join(OUT, f"hookspline_{base}.npz"), n=np.array(n), slots=np.array(slots),
                            src=np.array(src), E_uniform=Eu, x=x, v=v, X_psi=X1, V_psi=V1, X_tilde=X0, V_tilde=V0,
                            evals=np.array(ctx.field_evals))


def host_info():
    try:
        cpu = [l.split(":", 1)[1].strip() for l in open("/proc/cpuinfo") if l.startswith("model name")][0]
    except Exception:  # pragma: no cover
        cpu = platform.processor()
    import numba

    return dict(cpu=cpu, cores=os.cpu_count(), numba_threads=numba.config.NUMBA_NUM_THREADS,
                numpy=np.__version__, numba=numba.__version__, python=platform.python_version())


def main(argv):
    sys.path.insert(0, REF)
    names = argv or list(CONFIGS)
    for name in names:
        if name == "fields":
            field_goldens()
            continue
        if name == "checkpoints":
            checkpoint_goldens()
            continue
        if name == "hooks":
            hook_goldens()
            continue
        if name == "api":
            api_goldens()
            continue
        if name == "hooks_spline":
            hook_spline_goldens()
            continue
        if name.startswith("sweep_"):
            base = name[len("sweep_"):]
            g, ic = build(CONFIGS[base])
            z = np.load(os.path.join(OUT, f"{base}.npz"))
            stack = z["coeffs"].reshape((-1,) + (g.Nx,) * g.d)
            sweep_goldens(base, g, ic, stack, CONFIGS[base]["tau"])
            continue
        if name.startswith("trace_"):
            # trace goldens only, from the coefficients stored by an earlier run
            base = name[len("trace_"):]
            g, _ = build(CONFIGS[base])
            z = np.load(os.path.join(OUT, f"{base}.npz"))
            stack = z["coeffs"].reshape((-1,) + (g.Nx,) * g.d)
            trace_goldens(base, g, stack, CONFIGS[base]["tau"], TRACE_N[base])
            continue
        g, ic, hist = run(name, CONFIGS[name])
        if name in TRACE_N:
            trace_goldens(name, g, hist.stacked(), CONFIGS[name]["tau"], TRACE_N[name])


if __name__ == "__main__":
    main(sys.argv[1:])
