"""Per-rank work of the tensor-parallel configs on ONE GPU: a rank of TP=P
runs the block on a d_ff/P shard (balanced_ranges, tp.cpp:8-29), so its
kernel time is that of a (d_model, d_ff/P) block.  Times the library default,
the static plan with stage-1 split-K over a cluster, and the scheduler's pick,
with enough rotating weight sets that the working set is > 3x L2.

    python tools/tp_shard_sweep.py [--shapes llama8b,qwen32b,llama70b] [--batches 1,16,64]
"""
import argparse
import json
import math
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from paper_2602_11808_b200 import runtime as rt  # noqa: E402

SHAPES = {"llama8b": (4096, 14336, (1, 2, 4, 8)), "qwen7b": (3584, 18944, (1, 2, 4, 8)),
          "qwen32b": (5120, 27648, (1, 2, 4, 8)), "llama70b": (8192, 28672, (2, 4, 8))}

ap = argparse.ArgumentParser()
ap.add_argument("--shapes", default="llama8b,qwen32b,llama70b")
ap.add_argument("--batches", default="1,16,64")
ap.add_argument("--reps", type=int, default=30)
ap.add_argument("--specs", default="default;sk2;sk4;sk8;tune")
ap.add_argument("--json", default="")
ap.add_argument("--P", default="", help="comma list of TP degrees (default: per shape)")
a = ap.parse_args()
ctx = rt.Context(0)
peak = json.load(open("MEASURED_PEAKS.json"))["hbm_gbs"] if os.path.exists(
    "MEASURED_PEAKS.json") else 6650.0
ev0, ev1 = rt.Event(), rt.Event()
rows = []
for name in a.shapes.split(","):
    dm, df, Ps = SHAPES[name]
    if a.P:
        Ps = [int(v) for v in a.P.split(",")]
    for P in Ps:
        b0, b1 = rt.balanced_range(df, P, 0)
        dfs = b1 - b0
        wbytes = 3 * dm * dfs * 2
        nsets = max(2, math.ceil(3 * 126e6 / wbytes))
        s = 1 / np.sqrt(dm)
        sets = []
        for i in range(nsets):
            g = ctx.array((dm, dfs)).fill_uniform(10 * i + 1, -s, s)
            u = ctx.array((dm, dfs)).fill_uniform(10 * i + 2, -s, s)
            d = ctx.array((dfs, dm)).fill_uniform(10 * i + 3, -s, s)
            sets.append(ctx.weights(g, u, d))
            del g, u, d
        for B in [int(b) for b in a.batches.split(",")]:
            x = ctx.array((B, dm)).fill_uniform(5)
            y = ctx.array((B, dm), rt.F32)
            nbytes = 2 * (3 * dm * dfs + 2 * B * dm + 2 * B * dfs)
            res = {}
            for spec in a.specs.split(";"):
                if spec == "default":
                    cfg = None
                elif spec.startswith("sk"):
                    cfg = rt.Config.make(block_kernel=1, s1_split_k=int(spec[2:]))
                elif spec == "tune":
                    cfg, _, _ = ctx.tune(sets[0], B, None, 1, 4)
                else:
                    kw = {k: int(v) for k, v in (p.split("=") for p in spec.split(",") if p)}
                    cfg = rt.Config.make(**kw)
                try:
                    for i in range(2 * nsets):  # every set once (first-use costs)
                        ctx.forward(sets[i % nsets], x, y, cfg=cfg)
                    ctx.sync()
                    ev0.record(ctx)
                    for i in range(a.reps):
                        ctx.forward(sets[i % nsets], x, y, cfg=cfg)
                    ev1.record(ctx)
                    ctx.sync()
                    us = ev0.elapsed_ms(ev1) * 1e3 / a.reps
                except Exception as e:  # noqa: BLE001
                    print("ERR", name, P, B, spec, e, flush=True)
                    continue
                label = spec if spec != "tune" else "tune:" + cfg.label.decode()
                res[label] = us
                gbs = nbytes / us / 1e3
                rows.append({"shape": name, "P": P, "d_ff_shard": dfs, "B": B, "cfg": label,
                             "us": round(us, 2), "gbs": round(gbs, 1),
                             "frac": round(gbs / peak, 3)})
                print(f"{name:9s} P={P} dff/P={dfs:6d} B={B:3d} {label:45s} {us:8.2f} us "
                      f"{gbs:7.1f} GB/s  {gbs / peak:5.3f}", flush=True)
        del sets
if a.json:
    json.dump(rows, open(a.json, "w"), indent=1)
