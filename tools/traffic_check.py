"""One block call bracketed by cudaProfilerStart/Stop, for the ncu
traffic-model assertion (tests/test_traffic_ncu.py):

    ncu --profile-from-start off --metrics dram__bytes_read.sum,... --csv \\
        python tools/traffic_check.py --B 64 --variant fused
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from paper_2602_11808_b200 import runtime as rt  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--B", type=int, default=16)
ap.add_argument("--dm", type=int, default=4096)
ap.add_argument("--df", type=int, default=14336)
ap.add_argument("--variant", default="fused",
                choices=["fused", "fused_notail", "two", "four", "mutant2"])
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
cfg = {"fused": None, "two": rt.Config.make(variant=rt.VARIANT_TWO_KERNEL),
       "four": rt.Config.make(variant=rt.VARIANT_FOUR_KERNEL),
       # the fused block kernel with SiLU(A_gate) round-tripped through global
       # memory in its epilogue (MaterializeIntermediate, verification.cpp:126-169)
       "mutant2": rt.Config.make(block_kernel=1, dynamic_sched=1, mutant=2, s1_tail=1),
       # the default block kernel with whole stage-1 tiles only (no tail split:
       # every tile through the epilogue the mutant modifies)
       "fused_notail": rt.Config.make(block_kernel=1, dynamic_sched=1, s1_tail=1)}[a.variant]
for _ in range(3):
    ctx.forward(w, x, y, cfg=cfg)
ctx.profiler_range(True)
ctx.forward(w, x, y, cfg=cfg)
ctx.profiler_range(False)
print("done", flush=True)
