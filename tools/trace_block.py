"""Per-CTA timeline of one streaming-kernel launch (dfk_set_trace)."""
import argparse, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2602_11808_b200 import runtime as rt

ap = argparse.ArgumentParser()
ap.add_argument("--B", type=int, default=1)
ap.add_argument("--dm", type=int, default=4096)
ap.add_argument("--df", type=int, default=14336)
ap.add_argument("--cfgs", default="block:kbs=2;s1:kbs=3,s1_ctas=112;down:kbs=2")
a = ap.parse_args()
ctx = rt.Context(0)
DM, DF, B = a.dm, a.df, a.B
s = 1 / np.sqrt(DM)
sets = []
for i in range(3):
    g = ctx.array((DM, DF)).fill_uniform(10 * i + 1, -s, s)
    u = ctx.array((DM, DF)).fill_uniform(10 * i + 2, -s, s)
    d = ctx.array((DF, DM)).fill_uniform(10 * i + 3, -s, s)
    sets.append(ctx.weights(g, u, d)); del g, u, d
x = ctx.array((B, DM)).fill_uniform(5)
a2 = ctx.array((B, DF)); y = ctx.array((B, DM), rt.F32)
nsm = ctx.sm_count
tr = ctx.array((2 * nsm * 64,), rt.F32)  # 2*nsm*64 uint64 == 4*nsm*64 f32... sized below
tr = rt.DeviceArray(ctx, (2 * nsm * 64 * 2,), rt.F32)
for spec in a.cfgs.split(";"):
    kind, _, kv = spec.partition(":")
    kw = {k: int(v) for k, v in (p.split("=") for p in kv.split(",") if p)}
    if kind == "block":
        kw["block_kernel"] = 1
    cfg = rt.Config.make(**kw)
    def call(i):
        w = sets[i % 3]
        if kind == "s1":
            ctx.stage1(w, x, a2, cfg=cfg)
        elif kind == "down":
            ctx.down(w, a2, y, cfg=cfg)
        else:
            ctx.forward(w, x, y, cfg=cfg)
    for i in range(4):
        call(i)
    ctx.sync()
    tr.fill(0)
    ctx.set_trace(tr)
    call(5)
    ctx.sync()
    ctx.set_trace(None)
    raw = np.frombuffer(tr.download().tobytes(), dtype=np.uint64).reshape(-1, 64)
    used = raw[:, 0] > 0
    t = raw[used].astype(np.int64)
    t0 = t[:, 0].min()
    rel = np.where(t > 0, (t - t0) / 1000.0, np.nan)
    print(f"=== {spec}  (B={B}) CTAs={used.sum()}")
    print(f"  start  min/med/max  {np.nanmin(rel[:,0]):6.1f} {np.nanmedian(rel[:,0]):6.1f} {np.nanmax(rel[:,0]):6.1f} us")
    print(f"  prod done          {np.nanmin(rel[:,1]):6.1f} {np.nanmedian(rel[:,1]):6.1f} {np.nanmax(rel[:,1]):6.1f}")
    print(f"  cons done          {np.nanmin(rel[:,2]):6.1f} {np.nanmedian(rel[:,2]):6.1f} {np.nanmax(rel[:,2]):6.1f}")
    for i in range(6):
        iss, ret = rel[:, 3 + 2 * i], rel[:, 4 + 2 * i]
        if np.all(np.isnan(iss)):
            break
        n = np.sum(~np.isnan(ret))
        print(f"  piece {i}: n={n:3d} issue {np.nanmin(iss):6.1f} {np.nanmedian(iss):6.1f} {np.nanmax(iss):6.1f}"
              f"  retire {np.nanmin(ret):6.1f} {np.nanmedian(ret):6.1f} {np.nanmax(ret):6.1f}")
    if np.any(~np.isnan(rel[:, 61])):
        for sl, nm in ((61, "split: before wait"), (62, "split: after wait"), (63, "split: non-leader arrived")):
            col = rel[:, sl]
            lead = np.array([i % 4 == 0 for i in np.flatnonzero(used)])
            for who, m in (("leaders", lead), ("others", ~lead)):
                c = col[m]
                c = c[~np.isnan(c)]
                if len(c):
                    print(f"  {nm:28s} {who:8s} {c.min():6.1f} {np.median(c):6.1f} {c.max():6.1f}")
    if np.any(~np.isnan(rel[:, 44])):
        lead = np.array([i % 4 == 0 for i in np.flatnonzero(used)])
        for base, nm in ((44, "leader q: after wait"), (48, "leader q: after loop"), (52, "leader q: after arrives")):
            for qq in range(4):
                c = rel[lead, base + qq]
                c = c[~np.isnan(c)]
                if len(c):
                    print(f"  {nm} {qq}  {c.min():6.1f} {np.median(c):6.1f} {c.max():6.1f}")
    # coarse per-CTA listing of the slowest 5
    order = np.argsort(-rel[:, 2])[:8]
    for c in order:
        vals = " ".join(f"{v:6.1f}" for v in rel[c, 3:15] if not np.isnan(v))
        print(f"  cta{np.flatnonzero(used)[c]:4d} done {rel[c,2]:6.1f}: {vals}")
    sys.stdout.flush()
