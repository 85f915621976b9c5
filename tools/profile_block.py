"""Runs a few fused-block calls at Llama-8B shape for ncu capture.

    ncu --set full -k regex:stream_kernel -s 4 -c 2 -o prof python tools/profile_block.py --B 16
"""
import argparse, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2602_11808_b200 import runtime as rt

ap = argparse.ArgumentParser()
ap.add_argument("--B", type=int, default=16)
ap.add_argument("--dm", type=int, default=4096)
ap.add_argument("--df", type=int, default=14336)
ap.add_argument("--calls", type=int, default=6)
ap.add_argument("--family", default="tc", choices=["tc", "gemv"])
ap.add_argument("--variant", default="fused", choices=["fused", "two", "four"])
ap.add_argument("--s1-stages", type=int, default=0)
ap.add_argument("--pdl", type=int, default=1)
ap.add_argument("--path", default="default", choices=["default", "two", "block", "block-static"],
                help="default = the library's default config (NULL cfg)")
a = ap.parse_args()
ctx = rt.Context(0)
s = 1 / np.sqrt(a.dm)
g = ctx.array((a.dm, a.df)).fill_uniform(1, -s, s)
u = ctx.array((a.dm, a.df)).fill_uniform(2, -s, s)
d = ctx.array((a.df, a.dm)).fill_uniform(3, -s, s)
w = ctx.weights(g, u, d)
del g, u, d
x = ctx.array((a.B, a.dm)).fill_uniform(4)
y = ctx.array((a.B, a.dm), rt.F32)
fam = rt.FAMILY_TC if a.family == "tc" else rt.FAMILY_GEMV
var = {"fused": rt.VARIANT_FUSED, "two": rt.VARIANT_TWO_KERNEL, "four": rt.VARIANT_FOUR_KERNEL}[a.variant]
if a.path == "default" and a.variant == "fused":
    cfg = None
else:
    cfg = rt.Config.make(variant=var, s1_family=fam, down_family=fam, s1_stages=a.s1_stages,
                         pdl=a.pdl, block_kernel=int(a.path.startswith("block")),
                         dynamic_sched=int(a.path == "block"))
for i in range(a.calls):
    ctx.forward(w, x, y, cfg=cfg)
ctx.sync()
print("done", ctx.launch_count())
