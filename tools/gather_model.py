# Offline model of the d=1 shared-memory gather cost: bank-conflict wavefronts per 8-byte warp
# gather for x-fastest vs v-fastest lanes, from a ts1 history dumped by tools/dump_history.py.
import numpy as np, math
H = np.load('gpurun_out/ts1_hist.npy')  # (1601, 64)
N = 64; L = 4*math.pi; tau = 1/16; Nv = 512; vmax = 10.0
hx = L/N; hv = 2*vmax/Nv; inv_h = N/L
nodes = np.arange(N); vrows = np.arange(Nv)
x0 = (nodes*hx)[:, None] * np.ones((1, Nv))       # [node, row]
v0 = np.ones((N, 1)) * (-vmax + (vrows + 0.5)*hv)[None, :]
def E(c, x):
    u = np.mod(x, L); t = u*inv_h; i = np.minimum(t.astype(np.int64), N-1); f = t - i
    s = 1-f
    dw = [-0.5*s*s, f*(1.5*f-2), s*(2-1.5*s), 0.5*f*f]
    g = sum(c[(i + o - 1) % N]*dw[o] for o in range(4))
    return -g*inv_h, i
def wavefronts(cells):
    # cells: (32,) cell index per lane for an 8-byte gather; half-warps processed separately
    tot = 0
    for h in (cells[:16], cells[16:]):
        best = 1
        for b in range(16):
            d = np.unique(h[(h % 16) == b])
            best = max(best, len(d))
        tot += best
    return tot
for n in (100, 400, 800, 1200, 1600):
    x = x0.copy(); v = v0.copy()
    cells = []
    k = n
    while k > 1:
        k -= 1
        x = x - tau*v
        e, i = E(H[k], x); v = v + tau*e
        cells.append(i)
    x = x - tau*v; e, i = E(H[0], x); cells.append(i)
    cells = np.array(cells)  # (n, N, Nv)
    # sample substeps
    idx = np.linspace(0, n-1, 12).astype(int)
    wx = []; wv = []
    rng = np.random.default_rng(0)
    for s in idx:
        C = cells[s]
        for _ in range(40):
            j = rng.integers(Nv); t = rng.integers(2)
            wx.append(wavefronts(C[32*t:32*t+32, j]))        # lanes = 32 nodes, same v
            nd = rng.integers(N); r0 = 32*rng.integers(Nv//32)
            wv.append(wavefronts(C[nd, r0:r0+32]))          # lanes = 32 v rows, same node
    print(f"n={n}: x-fastest {np.mean(wx):.2f}  v-fastest {np.mean(wv):.2f} wavefronts per 8-byte gather")
