"""Per-block time of a decode chain (dfk_decode, CUDA graph) over TP-rank
shard shapes on one GPU: L distinct layers (> 3x L2 of weights in total),
`steps` passes.  (Used to A/B a next-layer L2 prefetch for small shards --
no gain, not kept: profiles/r1c_epilogue.md.)

    python tools/decode_shard_probe.py [--shapes ...] [--batches 1,16,64]
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from paper_2602_11808_b200 import runtime as rt  # noqa: E402

SHAPES = {"llama8b/8": (4096, 1792), "llama8b/4": (4096, 3584), "qwen32b/8": (5120, 3456),
          "llama70b/8": (8192, 3584), "llama8b/1": (4096, 14336), "qwen7b/1": (3584, 18944),
          "qwen32b/4": (5120, 6912), "qwen32b/2": (5120, 13824), "llama70b/4": (8192, 7168),
          "llama70b/2": (8192, 14336)}

ap = argparse.ArgumentParser()
ap.add_argument("--shapes", default="llama8b/8,llama8b/4,qwen32b/8,llama70b/8,llama8b/1")
ap.add_argument("--batches", default="1,16,64")
ap.add_argument("--steps", type=int, default=4)
a = ap.parse_args()
ctx = rt.Context(0)
ev0, ev1 = rt.Event(), rt.Event()
tag = os.environ.get("TAG", "")
for name in a.shapes.split(","):
    dm, df = SHAPES[name]
    L = max(4, int(np.ceil(3 * 126e6 / (6 * dm * df))))  # > 3x L2 of weights
    s = 1 / np.sqrt(dm)
    ws = []
    for l in range(L):
        g = ctx.array((dm, df)).fill_uniform(10 * l + 1, -s, s)
        u = ctx.array((dm, df)).fill_uniform(10 * l + 2, -s, s)
        d = ctx.array((df, dm)).fill_uniform(10 * l + 3, -s, s)
        ws.append(ctx.weights(g, u, d))
        del g, u, d
    for B in [int(v) for v in a.batches.split(",")]:
        x = ctx.array((B, dm)).fill_uniform(5)
        y = ctx.array((B, dm))
        for _ in range(2):
            ctx.decode(ws, x, a.steps, y)
        ctx.sync()
        reps = 5
        ev0.record(ctx)
        for _ in range(reps):
            ctx.decode(ws, x, a.steps, y)
        ev1.record(ctx)
        ctx.sync()
        us = ev0.elapsed_ms(ev1) * 1e3 / (reps * a.steps * L)
        gbs = 2 * (3 * dm * df + 2 * B * dm + 2 * B * df) / us / 1e3
        print(f"{tag} {name:11s} dm={dm} df={df} L={L} B={B:3d}  {us:7.2f} us/block  "
              f"{gbs:7.1f} GB/s", flush=True)
    del ws
