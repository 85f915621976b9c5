"""bench.py's e2e leg alone (host buffers through dfk_forward_host_async, one
host sync per step of the B sweep), for A/B of the host-copy pipeline:
    DFK_HOST_PIPE=0|1 python tools/e2e_probe.py"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2602_11808_b200 import runtime as rt
DM, DF, SWEEP = 4096, 14336, [1, 2, 4, 8, 16, 32, 64]
ctx = rt.Context(0)
s = 1 / np.sqrt(DM)
sets = []
for i in range(4):
    g = ctx.array((DM, DF)).fill_uniform(10 * i + 1, -s, s)
    u = ctx.array((DM, DF)).fill_uniform(10 * i + 2, -s, s)
    d = ctx.array((DF, DM)).fill_uniform(10 * i + 3, -s, s)
    sets.append(ctx.weights(g, u, d)); del g, u, d
hx = {B: rt.PinnedHost((B, DM), np.uint16) for B in SWEEP}
hy = {B: rt.PinnedHost((B, DM), np.float32) for B in SWEEP}
xs = {B: ctx.array((B, DM)).fill_uniform(7 + B) for B in SWEEP}
ys = {B: ctx.array((B, DM), rt.F32) for B in SWEEP}
for B in SWEEP:
    hx[B].arr[...] = xs[B].download_bits()
byts = sum(2 * (3 * DM * DF + 2 * B * DM + 2 * B * DF) for B in SWEEP)
def run(host, steps):
    for k in range(steps):
        for j, B in enumerate(SWEEP):
            w = sets[(k * len(SWEEP) + j) % 4]
            if host:
                ctx.forward_host_async(w, hx[B].arr, hy[B].arr)
            else:
                ctx.forward(w, xs[B], ys[B])
        ctx.sync()
for host in (False, True):
    run(host, 3)
    t0 = time.perf_counter(); run(host, 20); t = (time.perf_counter() - t0) / 20
    print(f"pipe={os.environ.get('DFK_HOST_PIPE', '1')} {'host ' if host else 'device'} "
          f"{t * 1e6:8.1f} us/step  {byts / t / 1e9:7.1f} GB/s", flush=True)
# per batch: 20 back-to-back calls, one sync
for B in SWEEP:
    res = []
    for host in (False, True):
        def go(n):
            for i in range(n):
                if host:
                    ctx.forward_host_async(sets[i % 4], hx[B].arr, hy[B].arr)
                else:
                    ctx.forward(sets[i % 4], xs[B], ys[B])
            ctx.sync()
        go(4)
        t0 = time.perf_counter(); go(20); res.append((time.perf_counter() - t0) / 20 * 1e6)
    print(f"  B={B:3d} device {res[0]:7.1f} us  host {res[1]:7.1f} us  (+{res[1] - res[0]:5.1f})", flush=True)
