"""Times the library-default fused block (NULL config) at Llama-8B shape for
A/B comparisons of two builds on the same box:
    DFK_LIB=abtest/libdfk_old.so python tools/ab_time.py
"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2602_11808_b200 import runtime as rt
DM, DF = 4096, 14336
ctx = rt.Context(0)
s = 1 / np.sqrt(DM)
sets = []
for i in range(4):
    g = ctx.array((DM, DF)).fill_uniform(10 * i + 1, -s, s)
    u = ctx.array((DM, DF)).fill_uniform(10 * i + 2, -s, s)
    d = ctx.array((DF, DM)).fill_uniform(10 * i + 3, -s, s)
    sets.append(ctx.weights(g, u, d)); del g, u, d
ev0, ev1 = rt.Event(), rt.Event()
out = []
for B in [int(v) for v in os.environ.get("AB_B", "1,16,64").split(",")]:
    x = ctx.array((B, DM)).fill_uniform(5); y = ctx.array((B, DM), rt.F32)
    for i in range(8):
        ctx.forward(sets[i % 4], x, y)
    ctx.sync(); ev0.record(ctx)
    for i in range(40):
        ctx.forward(sets[i % 4], x, y)
    ev1.record(ctx); ctx.sync()
    out.append(f"B={B}:{ev0.elapsed_ms(ev1) * 1e3 / 40:.2f}us")
print(os.environ.get("AB_TAG", os.environ.get("DFK_LIB", "new")), " ".join(out), flush=True)
