"""A/B of launch configurations of the stand-alone down kernel (dfk_down, the
reference's down_projection, swiglu.cpp:214-226) at Llama-8B shape with
rotating weight sets (> 3x L2):
    python tools/down_probe.py --batches 1,16,64 --specs "default;dynamic_sched=0"
"""
import argparse
import math
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
ap.add_argument("--specs", default="default")
a = ap.parse_args()
DM, DF = a.dm, a.df
ctx = rt.Context(0)
s = 1 / np.sqrt(DM)
NS = max(4, math.ceil(3 * 126e6 / (DM * DF * 2)))
sets = []
for i in range(NS):
    d = ctx.array((DF, DM)).fill_uniform(10 * i + 3, -s, s)
    sets.append(ctx.weights(None, None, d))
    del d
ev0, ev1 = rt.Event(), rt.Event()
for B in [int(v) for v in a.batches.split(",")]:
    a2 = ctx.array((B, DF)).fill_uniform(7)
    y = ctx.array((B, DM), rt.F32)
    nbytes = 2 * (B * DF + DF * DM + B * DM)
    for spec in a.specs.split(";"):
        kw = {k: int(v) for k, v in (p.split("=") for p in spec.split(",") if p and p != "default")}
        cfg = rt.Config.make(**kw) if kw else None
        for i in range(8):
            ctx.down(sets[i % NS], a2, y, cfg=cfg)
        ctx.sync()
        ev0.record(ctx)
        for i in range(a.reps):
            ctx.down(sets[i % NS], a2, y, cfg=cfg)
        ev1.record(ctx)
        ctx.sync()
        us = ev0.elapsed_ms(ev1) * 1e3 / a.reps
        print(f"down {DF}x{DM} B={B:3d} {spec:45s} {us:7.2f} us {nbytes / us / 1e3:7.1f} GB/s",
              flush=True)
