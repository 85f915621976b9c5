"""Quick GPU sanity run: tiny shapes through every family, printing errors."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import oracle
from paper_2602_11808_b200 import runtime as rt

o = oracle.Oracle()
ctx = rt.Context(0)
print("fingerprint", ctx.fingerprint(), flush=True)
def rel(a, b):
    return float(np.abs(np.asarray(a, np.float64) - b).max() / max(np.abs(b).max(), 1e-30))
for (B, dm, df) in [(1, 64, 64), (4, 128, 256), (16, 512, 1536), (3, 200, 300), (64, 1024, 2048)]:
    x, wu, wg, wd = o.make_instance(1, B, dm, df, 1 / np.sqrt(dm))
    x, wu, wg, wd = (o.quantize_bf16(a)[0] for a in (x, wu, wg, wd))
    a2r, yr = o.forward(x, wu, wg, wd)
    w = ctx.weights(wg, wu, wd)
    xd = ctx.array((B, dm)).upload(x)
    fams = [("tc", rt.FAMILY_TC)] + ([("gemv", rt.FAMILY_GEMV)] if B <= 8 else [])
    for name, fam in fams:
        cfg = rt.Config.make(s1_family=fam, down_family=fam)
        a2 = ctx.array((B, df)); y = ctx.array((B, dm), rt.F32)
        t = time.time()
        ctx.stage1(w, xd, a2, cfg=cfg); ctx.sync()
        e1 = rel(a2.download(), a2r)
        ctx.down(w, a2, y, cfg=cfg); ctx.sync()
        e2 = rel(y.download(), yr)
        print(f"B={B} dm={dm} df={df} {name}: a2 err {e1:.2e}  y err {e2:.2e}  ({time.time()-t:.2f}s)", flush=True)
    for v in (rt.VARIANT_TWO_KERNEL, rt.VARIANT_FOUR_KERNEL):
        y = ctx.array((B, dm), rt.F32)
        ctx.forward(w, xd, y, cfg=rt.Config.make(variant=v)); ctx.sync()
        print(f"   variant {v}: y err {rel(y.download(), yr):.2e}", flush=True)
print("done")
