"""Locates host-side blocking in dfk_decode under the emulated fused TP."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2602_11808_b200 import runtime as rt
mode = sys.argv[1]
P, B, dm, df = 2, 3, 384, 1000
if len(sys.argv) > 2:
    B, dm, df = (int(v) for v in sys.argv[2:5])
src = sys.argv[5] if len(sys.argv) > 5 else "dev"
ctxs = [rt.Context(0) for _ in range(P)]
for c in ctxs:
    c.tp_sym_create(8, dm)
rt.Context.tp_sym_attach(ctxs)
ws = []
for p, c in enumerate(ctxs):
    b, e = rt.balanced_range(df, P, p)
    lay = []
    for l in range(2):
        if src == "dev":
            g = c.array((dm, df)).fill_uniform(3 * l + 1, -0.05, 0.05)
            u = c.array((dm, df)).fill_uniform(3 * l + 2, -0.05, 0.05)
            d = c.array((df, dm)).fill_uniform(3 * l + 3, -0.05, 0.05)
        else:
            rng = np.random.default_rng(l)
            g, u = rng.uniform(-.05, .05, (dm, df)), rng.uniform(-.05, .05, (dm, df))
            d = rng.uniform(-.05, .05, (df, dm))
        lay.append(c.weights(g, u, d, ff_range=(b, e)))
    ws.append(lay)
xs = [c.array((B, dm)).fill_uniform(9) for c in ctxs]
yfs = [c.array((B, dm), rt.F32) for c in ctxs]
ys = [c.array((B, dm)) for c in ctxs]
for c in ctxs:
    c.sync()
t0 = time.time()
def log(m): print(f"{time.time() - t0:7.3f}s {m}", flush=True)
for it in range(3):
    for p, c in enumerate(ctxs):
        log(f"it{it} decode rank {p} mode {mode} ...")
        if mode == "fwd":
            c.tp_forward_fused(ws[p][0], xs[p], yfs[p])
        else:
            c.decode(ws[p], xs[p], 2, ys[p], graph=(mode == "graph"))
        log(f"it{it} decode rank {p} returned")
    for c in ctxs:
        c.sync()
    log(f"it{it} synced")
