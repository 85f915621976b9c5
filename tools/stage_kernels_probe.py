"""Time the separate stage-1 and down kernels (the reference API's
run_fused_stage1 and down_projection entry points, dfk_stage1 / dfk_down)
against their algorithmic bytes, Llama-8B shape, rotating weight sets:
    python tools/stage_kernels_probe.py [--batches 1,16,64]
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from paper_2602_11808_b200 import runtime as rt  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--batches", default="1,16,64")
ap.add_argument("--reps", type=int, default=40)
ap.add_argument("--dm", type=int, default=4096)
ap.add_argument("--df", type=int, default=14336)
a = ap.parse_args()
DM, DF = a.dm, a.df
ctx = rt.Context(0)
s = 1 / np.sqrt(DM)
import math
NS = max(4, math.ceil(3 * 126e6 / (3 * DM * DF * 2)))
sets = []
for i in range(NS):
    g = ctx.array((DM, DF)).fill_uniform(10 * i + 1, -s, s)
    u = ctx.array((DM, DF)).fill_uniform(10 * i + 2, -s, s)
    d = ctx.array((DF, DM)).fill_uniform(10 * i + 3, -s, s)
    sets.append(ctx.weights(g, u, d))
    del g, u, d
ev0, ev1 = rt.Event(), rt.Event()
for B in [int(v) for v in a.batches.split(",")]:
    x = ctx.array((B, DM)).fill_uniform(5)
    a2 = ctx.array((B, DF))
    y = ctx.array((B, DM), rt.F32)
    res = {}
    for name, fn, nbytes in (
            ("stage1", lambda w: ctx.stage1(w, x, a2), 2 * (B * DM + 2 * DM * DF + B * DF)),
            ("down", lambda w: ctx.down(w, a2, y), 2 * (B * DF + DF * DM + B * DM)),
            ("stage1+down", lambda w: (ctx.stage1(w, x, a2), ctx.down(w, a2, y)),
             2 * (B * DM + 2 * DM * DF + B * DF) + 2 * (B * DF + DF * DM + B * DM)),
            ("forward", lambda w: ctx.forward(w, x, y),
             2 * (B * DM + 2 * DM * DF + B * DF) + 2 * (B * DF + DF * DM + B * DM))):
        for i in range(8):
            fn(sets[i % NS])
        ctx.sync()
        ev0.record(ctx)
        for i in range(a.reps):
            fn(sets[i % NS])
        ev1.record(ctx)
        ctx.sync()
        us = ev0.elapsed_ms(ev1) * 1e3 / a.reps
        res[name] = f"{us:6.2f} us {nbytes / us / 1e3:7.1f} GB/s"
    print(f"{DM}x{DF} B={B:3d} " + " | ".join(f"{k}: {v}" for k, v in res.items()), flush=True)
