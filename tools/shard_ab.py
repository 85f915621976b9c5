"""A/B timing of the library-default fused block over TP-shard shapes, for
knob experiments (environment variables are read once per process, so run
one process per setting):

    AB_TAG=base python tools/shard_ab.py
    AB_TAG=kbs2 AB_CFG=block_kernel=1,dynamic_sched=1,kbs=2 python tools/shard_ab.py

Shapes: the per-rank blocks of BASELINE configs 4/5 and Llama-8B TP=8
(balanced_ranges shards), plus the full Llama-8B block.  Rotating weight
sets > 3x L2; PDL-chained back-to-back calls (µs per call, event-timed).
"""
import math
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from paper_2602_11808_b200 import runtime as rt  # noqa: E402

SHAPES = [(4096, 1792), (5120, 3456), (8192, 3584), (5120, 6912), (8192, 7168), (4096, 14336)]
shapes = SHAPES
if os.environ.get("AB_SHAPES"):
    shapes = [tuple(int(v) for v in s.split("x")) for s in os.environ["AB_SHAPES"].split(",")]
batches = [int(v) for v in os.environ.get("AB_B", "1,16,64").split(",")]
reps = int(os.environ.get("AB_REPS", "30"))
ctx = rt.Context(0)
kw = {k: int(v) for k, v in (p.split("=") for p in os.environ.get("AB_CFG", "").split(",") if p)}
cfg = rt.Config.make(**kw) if kw else None
ev0, ev1 = rt.Event(), rt.Event()
out = []
for dm, df in shapes:
    nsets = max(2, math.ceil(3 * 126e6 / (3 * dm * df * 2)))
    s = 1 / np.sqrt(dm)
    ws = []
    for i in range(nsets):
        g = ctx.array((dm, df)).fill_uniform(10 * i + 1, -s, s)
        u = ctx.array((dm, df)).fill_uniform(10 * i + 2, -s, s)
        d = ctx.array((df, dm)).fill_uniform(10 * i + 3, -s, s)
        ws.append(ctx.weights(g, u, d))
        del g, u, d
    cells = []
    for B in batches:
        x = ctx.array((B, dm)).fill_uniform(5)
        y = ctx.array((B, dm), rt.F32)
        for i in range(2 * nsets):
            ctx.forward(ws[i % nsets], x, y, cfg=cfg)
        ctx.sync()
        best = None
        for _ in range(3):
            ev0.record(ctx)
            for i in range(reps):
                ctx.forward(ws[i % nsets], x, y, cfg=cfg)
            ev1.record(ctx)
            ctx.sync()
            us = ev0.elapsed_ms(ev1) * 1e3 / reps
            best = us if best is None else min(best, us)
        cells.append(f"{best:6.2f}")
    out.append(f"{dm}x{df}:" + "/".join(cells))
    del ws
print(f"{os.environ.get('AB_TAG', 'run'):>10} " + "  ".join(out), flush=True)
