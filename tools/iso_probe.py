"""Isolated single-call latency (L2 flushed, no PDL partner) vs PDL-chained
per-call time of the default block kernel, Llama-8B shape, for A/B of launch
geometry knobs (DFK_GRID, ...):
    DFK_GRID=148 python tools/iso_probe.py
"""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from paper_2602_11808_b200 import runtime as rt  # noqa: E402

DM, DF = 4096, 14336
ctx = rt.Context(0)
s = 1 / np.sqrt(DM)
sets = []
for i in range(4):
    g = ctx.array((DM, DF)).fill_uniform(10 * i + 1, -s, s)
    u = ctx.array((DM, DF)).fill_uniform(10 * i + 2, -s, s)
    d = ctx.array((DF, DM)).fill_uniform(10 * i + 3, -s, s)
    sets.append(ctx.weights(g, u, d))
    del g, u, d
ev0, ev1 = rt.Event(), rt.Event()
out = []
for B in (1, 16, 64):
    x = ctx.array((B, DM)).fill_uniform(5)
    y = ctx.array((B, DM), rt.F32)
    for i in range(8):
        ctx.forward(sets[i % 4], x, y)
    ctx.sync()
    iso = []
    for i in range(9):
        ctx.flush_l2()
        ev0.record(ctx)
        ctx.forward(sets[i % 4], x, y)
        ev1.record(ctx)
        ctx.sync()
        iso.append(ev0.elapsed_ms(ev1) * 1e3)
    ev0.record(ctx)
    for i in range(40):
        ctx.forward(sets[i % 4], x, y)
    ev1.record(ctx)
    ctx.sync()
    out.append(f"B={B}: iso {statistics.median(iso):6.2f} chained {ev0.elapsed_ms(ev1) * 1e3 / 40:6.2f}")
print(os.environ.get("TAG", ""), " | ".join(out), flush=True)
