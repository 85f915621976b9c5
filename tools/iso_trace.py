import os, sys, numpy as np
sys.path.insert(0, '.')
from paper_2602_11808_b200 import runtime as rt
DM, DF = 4096, 14336
ctx = rt.Context(0)
s = 1/np.sqrt(DM)
sets = []
for i in range(2):
    g = ctx.array((DM, DF)).fill_uniform(10*i+1, -s, s); u = ctx.array((DM, DF)).fill_uniform(10*i+2, -s, s); d = ctx.array((DF, DM)).fill_uniform(10*i+3, -s, s)
    sets.append(ctx.weights(g, u, d)); del g, u, d
ev0, ev1 = rt.Event(), rt.Event()
buf = rt.DeviceArray(ctx, (ctx.sm_count * 64 * 4,), rt.F32)
for B in (1, 64):
    x = ctx.array((B, DM)).fill_uniform(5); y = ctx.array((B, DM), rt.F32)
    for i in range(6): ctx.forward(sets[i % 2], x, y)
    ctx.sync()
    for mode in ("iso", "chained"):
        buf.fill(0); ctx.sync()
        if mode == "iso":
            ctx.flush_l2(); ev0.record(ctx)
            ctx.set_trace(buf); ctx.forward(sets[0], x, y); ctx.set_trace(None)
            ev1.record(ctx); ctx.sync()
        else:
            for i in range(4): ctx.forward(sets[i % 2], x, y)
            ev0.record(ctx)
            ctx.set_trace(buf); ctx.forward(sets[0], x, y); ctx.set_trace(None)
            ctx.forward(sets[1], x, y); ev1.record(ctx); ctx.sync()
        raw = np.frombuffer(buf.download().tobytes(), dtype=np.uint64).reshape(-1, 64).astype(np.int64)
        raw = raw[raw[:, 0] > 0]
        t0 = raw[:, 0].min()
        st = (raw[:, 0] - t0) / 1e3; done = (raw[:, 2] - t0) / 1e3
        act = raw[:, 32]; act = (act[act > 0] - t0) / 1e3
        r1 = raw[:, 4]; r1 = (r1[r1 > 0] - t0) / 1e3
        print(f"B={B} {mode:8s} event {ev0.elapsed_ms(ev1)*1e3:7.2f} us  span {done.max():6.2f}  CTA start med {np.median(st):5.2f} max {st.max():5.2f}  first X load med {np.median(act):5.2f}  first piece retire med {np.median(r1):6.2f}  done min/med/max {done.min():6.2f}/{np.median(done):6.2f}/{done.max():6.2f}", flush=True)
