"""Per-piece timeline of one steady-state block-kernel launch: for every
piece a CTA took (stage-1 tile or down K chunk) the time its weights started
streaming, the time its activation loads could issue (down pieces: when the
stage-1 tiles it reads had published) and the time its accumulator retired.

    python tools/trace_pieces.py --B 64 [--cfg key=val,...] [--json out.json]

Per-CTA slots (kTraceSlots = 64, stream_kernels.cu): 0 CTA start, 3+2q issue
of piece q, 4+2q retire of piece q, 24+q piece descriptor
(down << 48 | nkb << 32 | tile), 32+q first activation load of piece q,
40+j / 52+j weight issue / full-barrier pass of ring stage DFK_TRACE_S0 + j.
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from paper_2602_11808_b200 import runtime as rt  # noqa: E402

KB_BYTES = 16384

ap = argparse.ArgumentParser()
ap.add_argument("--B", type=int, default=64)
ap.add_argument("--dm", type=int, default=4096)
ap.add_argument("--df", type=int, default=14336)
ap.add_argument("--cfg", default="")
ap.add_argument("--json", default="")
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
buf = rt.DeviceArray(ctx, (nsm * 64 * 4,), rt.F32)
for i in range(8):
    ctx.forward(sets[i % 4], x, y, cfg=cfg)
ctx.sync()
buf.fill(0)
ctx.sync()
for i in range(6):
    ctx.forward(sets[i % 4], x, y, cfg=cfg)
ctx.set_trace(buf)
ctx.forward(sets[2], x, y, cfg=cfg)
ctx.set_trace(None)
ctx.forward(sets[3], x, y, cfg=cfg)
ctx.sync()
raw = np.frombuffer(buf.download().tobytes(), dtype=np.uint64).reshape(-1, 64)
raw = raw[raw[:, 0] > 0]
t0 = int(raw[:, 0].min())
end = (int(raw[:, 2].max()) - t0) / 1e3

pieces = []
for c, r in enumerate(raw):
    prev_ret = None
    for q in range(8):
        iss, ret = int(r[3 + 2 * q]), int(r[4 + 2 * q])
        if iss == 0:
            break
        d = int(r[24 + q])
        act = int(r[32 + q])
        p = {"cta": c, "q": q, "down": (d >> 48) & 1, "nkb": (d >> 32) & 0xFFFF,
             "tile": d & 0xFFFFFFFF, "issue": (iss - t0) / 1e3,
             "act": (act - t0) / 1e3 if act else None,
             "retire": (ret - t0) / 1e3 if ret else None}
        # consumer time of this piece: from the previous retire (or the
        # first activation load) to this retire
        start = prev_ret if prev_ret is not None else p["act"]
        if p["retire"] is not None and start is not None:
            p["busy"] = p["retire"] - start
        prev_ret = p["retire"]
        pieces.append(p)


def summ(sel, label):
    if not sel:
        return
    busy = np.array([p["busy"] for p in sel if "busy" in p])
    mb = np.array([p["nkb"] * KB_BYTES / 1e6 for p in sel if "busy" in p])
    rate = mb / busy * 1e3  # GB/s per CTA
    waits = np.array([p["act"] - p["issue"] for p in sel if p["act"] is not None])
    print(f"{label}: n={len(sel)} nkb median {np.median([p['nkb'] for p in sel]):.0f}; "
          f"retire->retire us p10/med/p90 {np.percentile(busy, 10):.2f}/"
          f"{np.median(busy):.2f}/{np.percentile(busy, 90):.2f}; GB/s per CTA "
          f"p10/med/p90 {np.percentile(rate, 10):.1f}/{np.median(rate):.1f}/"
          f"{np.percentile(rate, 90):.1f}; act-issue lag us med/p90/max "
          f"{np.median(waits):.2f}/{np.percentile(waits, 90):.2f}/{waits.max():.2f}")


print(f"B={B} cfg={a.cfg or 'default'} CTAs={len(raw)} launch span {end:.1f} us")
s1 = [p for p in pieces if not p["down"]]
dn = [p for p in pieces if p["down"]]
summ(s1, "stage-1 pieces")
summ(dn, "down pieces   ")
s1_last = max(p["retire"] for p in s1 if p["retire"] is not None)
print(f"last stage-1 retire {s1_last:.1f} us; first down act-load "
      f"{min(p['act'] for p in dn if p['act'] is not None):.1f} us")
# Time each CTA spends between its last retire and the launch end (tail).
last = np.array([max(p["retire"] for p in pieces if p["cta"] == c and p["retire"])
                 for c in range(len(raw))])
print(f"CTA finish us p10/med/p90/max {np.percentile(last, 10):.1f}/"
      f"{np.median(last):.1f}/{np.percentile(last, 90):.1f}/{last.max():.1f}")
# Down-phase stall: per down piece, time between weight issue and act issue.
hist = np.histogram([p["act"] for p in dn if p["act"] is not None],
                    bins=np.linspace(0, end, 11))[0]
print("down act-load issue histogram over the launch (10 bins):", hist.tolist())
per_cta = {}
for p in pieces:
    per_cta.setdefault(p["cta"], []).append(("D" if p["down"] else "S") + str(p["nkb"]))
shapes = {}
for v in per_cta.values():
    k = " ".join(v)
    shapes[k] = shapes.get(k, 0) + 1
print("piece sequences (count: seq):")
for k, n in sorted(shapes.items(), key=lambda kv: -kv[1])[:8]:
    print(f"  {n:3d}: {k}")
if a.json:
    with open(a.json, "w") as f:
        json.dump({"B": B, "span_us": end, "t0": t0, "pieces": pieces,
                   "raw": [[(int(v) - t0) if 0 < int(v) and i not in range(24, 32)
                            else int(v) for i, v in enumerate(r)] for r in raw]}, f)
# Ring stages kTraceStage0 .. +11 (stream_kernels.cu): weight issue (40+i)
# and full-barrier completion (52+i) -> per-stage landing latency and the
# spacing of completions (the CTA's streaming rate).
if int(os.environ.get("DFK_TRACE_S0", 24)) < 0:
    # first down piece of each CTA: 40 accumulator ready, 41/42 red.adds
    # issued (+ CTA barrier), 43 counter atom.acq_rel returned (its release
    # MEMBAR included), 44 finish done (finalize when last), 45 = 1 if this
    # CTA finalized
    d = raw[:, 40:46].astype(np.int64)
    okd = (d[:, :5] > 0).all(1)
    if okd.any():
        d = d[okd]
        med = lambda x: np.median(x) / 1e3
        fin = d[:, 5] == 1
        print(f"down epilogue (first down piece, {int(okd.sum())} CTAs, median us): reds+bar "
              f"{med(d[:, 1] - d[:, 0]):.2f}, fence {med(d[:, 2] - d[:, 1]):.2f}, atomic "
              f"{med(d[:, 3] - d[:, 2]):.2f}, finish {med(d[:, 4] - d[:, 3]):.2f} "
              f"(finalizing CTAs {int(fin.sum())}: "
              f"{(np.median(d[fin, 4] - d[fin, 3]) / 1e3) if fin.any() else 0:.2f})")
    # first piece when it is a stage-1 stream-K piece: 52 accumulator ready,
    # 46/47 red.adds issued (+ barrier), 48 counter atom.acq_rel returned,
    # 49 finalize done, 50 published (finalizing CTAs), 51 = 1 if finalized
    e = raw[:, [52, 46, 47, 48, 49, 50, 51]].astype(np.int64)
    oke = (e[:, :4] > 0).all(1)
    if oke.any():
        e = e[oke]
        fin = e[:, 6] == 1
        med = lambda x: np.median(x) / 1e3 if len(x) else 0.0
        print(f"stage-1 stream-K epilogue (first piece, {int(oke.sum())} CTAs, median us): "
              f"reds+bar {med(e[:, 1] - e[:, 0]):.2f}, fence {med(e[:, 2] - e[:, 1]):.2f}, "
              f"atomic {med(e[:, 3] - e[:, 2]):.2f}; finalizing CTAs {int(fin.sum())}: "
              f"finalize {med(e[fin, 4] - e[fin, 3]):.2f}, publish {med(e[fin, 5] - e[fin, 4]):.2f}")
    sys.exit(0)
iss = raw[:, 40:52].astype(np.int64)
ful = raw[:, 52:64].astype(np.int64)
nst = int(((iss > 0) & (ful > 0)).all(0).sum())  # stages every CTA traced
iss, ful = iss[:, :max(nst, 2)], ful[:, :max(nst, 2)]
ok = (iss > 0).all(1) & (ful > 0).all(1)
if not ok.any():
    print("ring stages: none traced on every CTA (pieces shorter than DFK_TRACE_S0 + 2)")
    sys.exit(0)
lat = (ful[ok] - iss[ok]) / 1e3
gap = np.diff(ful[ok], axis=1) / 1e3
print(f"ring stages {os.environ.get('DFK_TRACE_S0', 24)}+0..{nst - 1} on {int(ok.sum())} CTAs: issue->full latency us "
      f"p10/med/p90 {np.percentile(lat, 10):.2f}/{np.median(lat):.2f}/"
      f"{np.percentile(lat, 90):.2f}; full->full spacing us p10/med/p90 "
      f"{np.percentile(gap, 10):.2f}/{np.median(gap):.2f}/{np.percentile(gap, 90):.2f}")
ep = raw[:, 19:23].astype(np.int64)
okp = (ep > 0).all(1)
if okp.any():
    e = ep[okp]
    mma_end = None
    print(f"stage-1 epilogue of piece 0 on {int(okp.sum())} CTAs (us, median): "
          f"tfull->smem staged {np.median(e[:, 1] - e[:, 0]) / 1e3:.2f}, "
          f"TMA store + wait {np.median(e[:, 2] - e[:, 1]) / 1e3:.2f}, "
          f"fence + flag {np.median(e[:, 3] - e[:, 2]) / 1e3:.2f}; "
          f"tfull at {np.median(e[:, 0] - raw[okp, 32].astype(np.int64)) / 1e3:.1f} us "
          f"after the first activation load")
e2 = raw[:, [19, 23, 31, 20]].astype(np.int64)
ok2 = (e2 > 0).all(1)
if ok2.any():
    e2 = e2[ok2]
    print(f"  tfull->first TMEM load done {np.median(e2[:, 1] - e2[:, 0]) / 1e3:.2f}, "
          f"-> loop done {np.median(e2[:, 2] - e2[:, 1]) / 1e3:.2f}, "
          f"-> staged (named barrier) {np.median(e2[:, 3] - e2[:, 2]) / 1e3:.2f} us")
