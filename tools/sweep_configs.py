"""Times stage-1 / down / block / full-forward launch configurations at the
Llama-8B shape (rotating weight sets, CUDA events) — for tuning the kernels."""
import argparse, itertools, json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2602_11808_b200 import runtime as rt

ap = argparse.ArgumentParser()
ap.add_argument("--dm", type=int, default=4096)
ap.add_argument("--df", type=int, default=14336)
ap.add_argument("--batches", default="1,16,64")
ap.add_argument("--sets", type=int, default=3)
ap.add_argument("--reps", type=int, default=20)
ap.add_argument("--what", default="s1,down,block,fwd")
ap.add_argument("--specs", default="", help="';'-separated kind:k=v,... (kind s1|down|block|fwd|two)")
a = ap.parse_args()
DM, DF = a.dm, a.df
ctx = rt.Context(0)
s = 1 / np.sqrt(DM)
sets = []
for i in range(a.sets):
    g = ctx.array((DM, DF)).fill_uniform(10 * i + 1, -s, s)
    u = ctx.array((DM, DF)).fill_uniform(10 * i + 2, -s, s)
    d = ctx.array((DF, DM)).fill_uniform(10 * i + 3, -s, s)
    sets.append(ctx.weights(g, u, d)); del g, u, d
ev0, ev1 = rt.Event(), rt.Event()
def timeit(fn):
    for i in range(3): fn(i)
    ctx.sync(); ev0.record(ctx)
    for i in range(a.reps): fn(i)
    ev1.record(ctx); ctx.sync()
    return ev0.elapsed_ms(ev1) * 1e3 / a.reps
s1b = lambda B: 2 * (B * DM + 2 * DM * DF + B * DF)
dnb = lambda B: 2 * (B * DF + DF * DM + B * DM)
what = a.what.split(",")
for B in [int(b) for b in a.batches.split(",")]:
    x = ctx.array((B, DM)).fill_uniform(5)
    a2 = ctx.array((B, DF))
    y = ctx.array((B, DM), rt.F32)
    fams = [rt.FAMILY_TC] + ([rt.FAMILY_GEMV] if B <= 8 else [])
    res = []
    if "s1" in what:
        for fam, kbs, st, ctas in itertools.product(fams, (2, 3, 4), (0,), (0, 112)):
            cfg = rt.Config.make(s1_family=fam, kbs=kbs, s1_stages=st, s1_ctas=ctas)
            try:
                us = timeit(lambda i: ctx.stage1(sets[i % len(sets)], x, a2, cfg=cfg))
            except Exception as e:
                print("ERR", e); continue
            res.append(("s1", fam, kbs, st, ctas, us, s1b(B) / us / 1e3))
    if "down" in what:
        ctx.stage1(sets[0], x, a2)
        for fam, kbs, st, ctas in itertools.product(fams, (2, 3, 4), (0,), (74, 96, 112, 0)):
            cfg = rt.Config.make(down_family=fam, kbs=kbs, down_stages=st, down_ctas=ctas)
            us = timeit(lambda i: ctx.down(sets[i % len(sets)], a2, y, cfg=cfg))
            res.append(("down", fam, kbs, st, ctas, us, dnb(B) / us / 1e3))
    if "block" in what:
        for fam, kbs, st in itertools.product(fams, (2, 3, 4), (0,)):
            cfg = rt.Config.make(block_kernel=1, s1_family=fam, down_family=fam, kbs=kbs, s1_stages=st)
            us = timeit(lambda i: ctx.forward(sets[i % len(sets)], x, y, cfg=cfg))
            res.append(("block", fam, kbs, st, 0, us, (s1b(B) + dnb(B)) / us / 1e3))
    if "fwd" in what:
        for fam, kbs, pdl in itertools.product(fams, (2, 3), (1,)):
            cfg = rt.Config.make(s1_family=fam, down_family=rt.FAMILY_TC, kbs=kbs, pdl=pdl)
            us = timeit(lambda i: ctx.forward(sets[i % len(sets)], x, y, cfg=cfg))
            res.append(("fwd", fam, kbs, pdl, 0, us, (s1b(B) + dnb(B)) / us / 1e3))
        for v in (rt.VARIANT_TWO_KERNEL,):
            cfg = rt.Config.make(variant=v)
            us = timeit(lambda i: ctx.forward(sets[i % len(sets)], x, y, cfg=cfg))
            res.append(("cublas", 0, 0, 0, 0, us, (s1b(B) + dnb(B)) / us / 1e3))
    for spec in [t for t in a.specs.split(";") if t]:
        kind, _, kv = spec.partition(":")
        kw = {k: int(v) for k, v in (p.split("=") for p in kv.split(",") if p)}
        if kind == "block":
            kw["block_kernel"] = 1
        if kind == "two":
            kw["variant"] = rt.VARIANT_TWO_KERNEL
        cfg = rt.Config.make(**kw)
        if kind == "s1":
            fn, nb = (lambda i: ctx.stage1(sets[i % len(sets)], x, a2, cfg=cfg)), s1b(B)
        elif kind == "down":
            ctx.stage1(sets[0], x, a2)
            fn, nb = (lambda i: ctx.down(sets[i % len(sets)], a2, y, cfg=cfg)), dnb(B)
        else:
            fn, nb = (lambda i: ctx.forward(sets[i % len(sets)], x, y, cfg=cfg)), s1b(B) + dnb(B)
        us = timeit(fn)
        res.append((kind, kv, "", "", 0, us, nb / us / 1e3))
    print(f"=== B={B}")
    for r in res:
        if isinstance(r[1], str):
            print(f"  {r[0]:6s} {r[1]:40s}  {r[5]:8.2f} us  {r[6]:7.1f} GB/s")
        else:
            print(f"  {r[0]:6s} fam={r[1]} kbs={r[2]} st={r[3]} ctas={r[4]:3d}  {r[5]:8.2f} us  {r[6]:7.1f} GB/s")
    sys.stdout.flush()
