"""Warp-GEMV family vs tcgen05 (dynamic block kernel) at small batches over
full and TP-shard shapes, for A/B of two builds (DFK_LIB=...):
    DFK_LIB=abtest/libdfk_old.so python tools/gemv_ab.py
"""
import math
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from paper_2602_11808_b200 import runtime as rt  # noqa: E402

SHAPES = [("llama8b", 4096, 14336), ("llama8b/8", 4096, 1792), ("qwen32b/8", 5120, 3456),
          ("llama70b/8", 8192, 3584), ("qwen32b/4", 5120, 6912)]
ctx = rt.Context(0)
ev0, ev1 = rt.Event(), rt.Event()
tag = os.environ.get("TAG", os.environ.get("DFK_LIB", "cur"))
for name, dm, df in SHAPES:
    nsets = max(2, math.ceil(3 * 126e6 / (3 * dm * df * 2)))
    s = 1 / np.sqrt(dm)
    sets = []
    for i in range(nsets):
        g = ctx.array((dm, df)).fill_uniform(10 * i + 1, -s, s)
        u = ctx.array((dm, df)).fill_uniform(10 * i + 2, -s, s)
        d = ctx.array((df, dm)).fill_uniform(10 * i + 3, -s, s)
        sets.append(ctx.weights(g, u, d))
        del g, u, d
    out = []
    for B in (1, 2, 4):
        x = ctx.array((B, dm)).fill_uniform(5)
        y = ctx.array((B, dm), rt.F32)
        for fam, lab in ((rt.FAMILY_GEMV, "gemv"), (rt.FAMILY_TC, "tc")):
            cfg = rt.Config.make(s1_family=fam, down_family=fam, block_kernel=1, dynamic_sched=1)
            for i in range(2 * nsets):
                ctx.forward(sets[i % nsets], x, y, cfg=cfg)
            ctx.sync()
            ev0.record(ctx)
            for i in range(30):
                ctx.forward(sets[i % nsets], x, y, cfg=cfg)
            ev1.record(ctx)
            ctx.sync()
            out.append(f"B{B}-{lab} {ev0.elapsed_ms(ev1) * 1e3 / 30:6.2f}")
    print(f"{tag:24s} {name:11s} " + "  ".join(out), flush=True)
    del sets
