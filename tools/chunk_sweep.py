"""Sweep of the dynamic block kernel's work-split parameters over the
tensor-parallel shard shapes (BASELINE configs 2-5 at TP = 2/4/8): stage-1
stream-K chunk (s1_chunk_kb), down chunk (chunk_kb) and kernel family, per
batch, against the library default -- the data the default heuristics in
api.cu (fill_dynamic, default_config) are fitted to.

    python tools/chunk_sweep.py --json out.json [--shapes ...] [--batches ...]
"""
import argparse
import json
import math
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from paper_2602_11808_b200 import runtime as rt  # noqa: E402

SHAPES = {"llama8b": (4096, 14336), "qwen7b": (3584, 18944), "qwen32b": (5120, 27648),
          "llama70b": (8192, 28672)}

ap = argparse.ArgumentParser()
ap.add_argument("--shapes", default="llama8b:2,4,8;qwen7b:2,4,8;qwen32b:2,4,8;llama70b:2,4,8")
ap.add_argument("--batches", default="1,2,4,8,16,32,64")
ap.add_argument("--reps", type=int, default=30)
ap.add_argument("--json", default="")
ap.add_argument("--cks", default="0,8,16", help="down chunk sizes (0 = heuristic)")
a = ap.parse_args()
ctx = rt.Context(0)
ev0, ev1 = rt.Event(), rt.Event()
rows = []


def timeit(sets, x, y, cfg, reps):
    n = len(sets)
    for i in range(2 * n):
        ctx.forward(sets[i % n], x, y, cfg=cfg)
    ctx.sync()
    ev0.record(ctx)
    for i in range(reps):
        ctx.forward(sets[i % n], x, y, cfg=cfg)
    ev1.record(ctx)
    ctx.sync()
    return ev0.elapsed_ms(ev1) * 1e3 / reps


for spec in a.shapes.split(";"):
    name, Ps = spec.split(":")
    dm, df = SHAPES[name]
    for P in (int(v) for v in Ps.split(",")):
        b0, b1 = rt.balanced_range(df, P, 0)
        dfs = b1 - b0
        nsets = max(2, math.ceil(3 * 126e6 / (3 * dm * dfs * 2)))
        s = 1 / np.sqrt(dm)
        sets = []
        for i in range(nsets):
            g = ctx.array((dm, dfs)).fill_uniform(10 * i + 1, -s, s)
            u = ctx.array((dm, dfs)).fill_uniform(10 * i + 2, -s, s)
            d = ctx.array((dfs, dm)).fill_uniform(10 * i + 3, -s, s)
            sets.append(ctx.weights(g, u, d))
            del g, u, d
        kb1 = dm // 64
        t1 = (dfs + 63) // 64
        s1ks = sorted({16, 20, 24, 27, 32, 40, 48, 64, kb1} & set(range(16, kb1 + 1)))
        for B in (int(v) for v in a.batches.split(",")):
            x = ctx.array((B, dm)).fill_uniform(5)
            y = ctx.array((B, dm), rt.F32)
            nbytes = 2 * (3 * dm * dfs + 2 * B * dm + 2 * B * dfs)
            cfgs = {"default": None}
            fams = [rt.FAMILY_TC] + ([rt.FAMILY_GEMV] if B <= 8 else [])
            for fam in fams:
                for s1k in s1ks:
                    for ck in (int(v) for v in a.cks.split(",")):
                        lab = f"{'gemv' if fam == rt.FAMILY_GEMV else 'tc'}_s1k{s1k}_ck{ck}"
                        cfgs[lab] = rt.Config.make(s1_family=fam, down_family=fam,
                                                   block_kernel=1, dynamic_sched=1,
                                                   s1_chunk_kb=s1k, chunk_kb=ck)
            cfgs["cublaslt"] = rt.Config.make(variant=rt.VARIANT_TWO_KERNEL)
            res = {}
            for lab, cfg in cfgs.items():
                try:
                    res[lab] = round(timeit(sets, x, y, cfg, a.reps), 2)
                except Exception as e:  # noqa: BLE001
                    print("ERR", name, P, B, lab, e, flush=True)
            best = min((v, k) for k, v in res.items())
            rows.append({"shape": name, "P": P, "d_model": dm, "d_ff_shard": dfs, "t1": t1,
                         "kb1": kb1, "B": B, "bytes": nbytes, "us": res})
            print(f"{name:9s} P={P} t1={t1:4d} kb1={kb1:4d} B={B:3d} default {res['default']:7.2f}"
                  f"  best {best[1]:22s} {best[0]:7.2f}  cublaslt {res.get('cublaslt', 0):7.2f}",
                  flush=True)
        del sets
        if a.json:
            json.dump(rows, open(a.json, "w"))
