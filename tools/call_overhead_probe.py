"""Host-side cost of one forward call (C ABI through ctypes) and the latency
of a single synchronised call, device buffers vs host buffers (Llama-8B, B=16):
    python tools/call_overhead_probe.py
Measured (B200, r1c): submit 7.2 us/call device path, 13.9 us/call host path
(H2D + D2H on side streams with flag waits); one synchronised call 72.6 /
91.4 us against a ~53 us kernel.
"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2602_11808_b200 import runtime as rt
ctx = rt.Context(0)
DM, DF = 4096, 14336
s = 1 / np.sqrt(DM)
g = ctx.array((DM, DF)).fill_uniform(1, -s, s); u = ctx.array((DM, DF)).fill_uniform(2, -s, s); d = ctx.array((DF, DM)).fill_uniform(3, -s, s)
w = ctx.weights(g, u, d)
x = ctx.array((16, DM)).fill_uniform(5); y = ctx.array((16, DM), rt.F32)
hx = rt.PinnedHost((16, DM), np.uint16); hy = rt.PinnedHost((16, DM), np.float32)
for _ in range(20): ctx.forward(w, x, y)
ctx.sync()
N = 200
t0 = time.perf_counter()
for _ in range(N): ctx.forward(w, x, y)
t1 = time.perf_counter(); ctx.sync(); t2 = time.perf_counter()
print(f"device path: host submit {(t1-t0)/N*1e6:.2f} us/call, total {(t2-t0)/N*1e6:.2f} us/call")
for _ in range(20): ctx.forward_host_async(w, hx.arr, hy.arr)
ctx.sync()
t0 = time.perf_counter()
for _ in range(N): ctx.forward_host_async(w, hx.arr, hy.arr)
t1 = time.perf_counter(); ctx.sync(); t2 = time.perf_counter()
print(f"host path: host submit {(t1-t0)/N*1e6:.2f} us/call, total {(t2-t0)/N*1e6:.2f} us/call")
# first-call latency after sync: time from submit to completion of a single call
lat = []
for _ in range(20):
    ctx.sync(); t0 = time.perf_counter(); ctx.forward(w, x, y); ctx.sync(); lat.append(time.perf_counter() - t0)
print(f"single device call incl. sync: {np.median(lat)*1e6:.1f} us")
lat = []
for _ in range(20):
    ctx.sync(); t0 = time.perf_counter(); ctx.forward_host_async(w, hx.arr, hy.arr); ctx.sync(); lat.append(time.perf_counter() - t0)
print(f"single host-buffer call incl. sync: {np.median(lat)*1e6:.1f} us")
