"""Steady-state timeline of consecutive block-kernel launches (PDL-chained,
no host sync between them): each launch writes its own trace buffer
(dfk_set_trace is latched at launch time), all stamps are globaltimer, so the
tail of launch i and the ramp of launch i+1 line up.

    python tools/trace_pair.py --B 1 [--n 3] [--cfg key=val,...]
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from paper_2602_11808_b200 import runtime as rt  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--B", type=int, default=1)
ap.add_argument("--dm", type=int, default=4096)
ap.add_argument("--df", type=int, default=14336)
ap.add_argument("--n", type=int, default=3)
ap.add_argument("--cfg", default="")
a = ap.parse_args()
ctx = rt.Context(0)
DM, DF, B = a.dm, a.df, a.B
s = 1 / np.sqrt(DM)
sets = []
for i in range(4):
    g = ctx.array((DM, DF)).fill_uniform(10 * i + 1, -s, s)
    u = ctx.array((DM, DF)).fill_uniform(10 * i + 2, -s, s)
    d = ctx.array((DF, DM)).fill_uniform(10 * i + 3, -s, s)
    sets.append(ctx.weights(g, u, d))
    del g, u, d
x = ctx.array((B, DM)).fill_uniform(5)
y = ctx.array((B, DM), rt.F32)
kw = {k: int(v) for k, v in (p.split("=") for p in a.cfg.split(",") if p)}
cfg = rt.Config.make(**kw) if kw else None
nsm = ctx.sm_count
bufs = [rt.DeviceArray(ctx, (nsm * 64 * 4,), rt.F32) for _ in range(a.n)]
for i in range(8):
    ctx.forward(sets[i % 4], x, y, cfg=cfg)
ctx.sync()
for b in bufs:
    b.fill(0)
ctx.sync()
for i in range(6):  # keep the pipeline busy before the traced launches
    ctx.forward(sets[i % 4], x, y, cfg=cfg)
for i, b in enumerate(bufs):
    ctx.set_trace(b)
    ctx.forward(sets[(6 + i) % 4], x, y, cfg=cfg)
ctx.set_trace(None)
ctx.forward(sets[0], x, y, cfg=cfg)
ctx.sync()
tabs = []
for b in bufs:
    raw = np.frombuffer(b.download().tobytes(), dtype=np.uint64).reshape(-1, 64)
    tabs.append(raw[raw[:, 0] > 0].astype(np.int64))
t0 = tabs[0][:, 0].min()


def q(v):
    v = v[v > 0]
    r = (v - t0) / 1000.0
    return f"{r.min():7.1f} {np.percentile(r, 10):7.1f} {np.median(r):7.1f} " \
           f"{np.percentile(r, 90):7.1f} {r.max():7.1f}"


print(f"B={B} cfg={a.cfg or 'default'}  columns: min p10 median p90 max (us from launch 0 start)")
for i, t in enumerate(tabs):
    print(f"launch {i}: CTAs={len(t)}")
    print(f"  cta start      {q(t[:, 0])}")
    print(f"  first issue    {q(t[:, 3])}")
    print(f"  first retire   {q(t[:, 4])}")
    print(f"  producer done  {q(t[:, 1])}")
    print(f"  consumer done  {q(t[:, 2])}")
    if i:
        prev_end = (tabs[i - 1][:, 2].max() - t0) / 1000.0
        start = (t[:, 0] - t0) / 1000.0
        print(f"  CTAs started before the previous launch's last CTA finished: "
              f"{int(np.sum(start < prev_end))}; launch period "
              f"{(t[:, 2].max() - tabs[i - 1][:, 2].max()) / 1000.0:.1f} us")
    for k in range(8):
        iss, ret = t[:, 3 + 2 * k], t[:, 4 + 2 * k]
        if not np.any(iss > 0):
            break
        print(f"  piece {k}: n={int(np.sum(ret > 0)):3d} issue {q(iss)}  retire {q(ret)}")
