"""Child of tests/test_gpu_sanitizer.py: small instances of every block-kernel
schedule (run under compute-sanitizer), each checked against the oracle."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle  # noqa: E402
from paper_2602_11808_b200 import runtime as rt  # noqa: E402

orc = oracle.Oracle()


def inst(seed, B, dm, df):
    return tuple(orc.quantize_bf16(a)[0] for a in orc.make_instance(seed, B, dm, df, dm ** -0.5))


def check(y, ref, what):
    err = float(np.abs(y - ref).max() / np.abs(ref).max())
    assert err <= 1e-2, (what, err)


ctx = rt.Context(0)
# full stage-1 wave is too big for the sanitizer; small shards exercise the
# stream-K stage 1, the dynamic queue, the A2 flags and the down counters
cases = {
    "default": None,
    "s1_stream_k": rt.Config.make(block_kernel=1, dynamic_sched=1, s1_chunk_kb=2),
    "split_k_cluster": rt.Config.make(block_kernel=1, s1_split_k=2),
    "static_block": rt.Config.make(block_kernel=1),
    "two_kernel_fused": rt.Config.make(),
}
for B in (3, 33):
    x, wu, wg, wd = inst(7 + B, B, 256, 640)
    _, ref = orc.forward(x, wu, wg, wd)
    w = ctx.weights(wg, wu, wd)
    xd = ctx.array((B, 256)).upload(x)
    y = ctx.array((B, 256), rt.F32)
    for name, cfg in cases.items():
        for _ in range(2):
            ctx.forward(w, xd, y, cfg=cfg)
        check(y.download(), ref, (name, B))
# emulated fused TP all-reduce: 2 ranks as 2 contexts on this GPU
P, B, dm, df = 2, 5, 256, 700
x, wu, wg, wd = inst(99, B, dm, df)
_, ref = orc.forward(x, wu, wg, wd)
ctxs = [rt.Context(0) for _ in range(P)]
for c in ctxs:
    c.tp_sym_create(8, dm)
rt.Context.tp_sym_attach(ctxs)
ws, xs, ys = [], [], []
for p, c in enumerate(ctxs):
    b, e = rt.balanced_range(df, P, p)
    ws.append(c.weights(wg, wu, wd, ff_range=(b, e)))
    xs.append(c.array((B, dm)).upload(x))
    ys.append(c.array((B, dm), rt.F32))
for _ in range(2):
    for p, c in enumerate(ctxs):
        c.tp_forward_fused(ws[p], xs[p], ys[p])
    for c in ctxs:
        c.sync()
for p in range(P):
    check(ys[p].download(), ref, ("fused_tp", p))
print("sanitizer child ok")
