"""Lifetime and protocol contracts of the captured decode graphs and the fused
tensor-parallel all-reduce (single process; ranks emulated by several
contexts on one GPU):

* a captured graph stays correct after scratch buffers are reallocated by a
  larger call (the graph bakes addresses in: it must be re-captured);
* a graph over layers whose stage-1 tile counts differ replays correctly
  with new inputs (per-tile completion flags must not leak across replays);
* the GEMV family's 8-row chunks through the host-buffer path and the fused
  all-reduce (B = 9..16);
* the fused all-reduce writes Y (fp32 or bf16) itself -- one launch per
  block -- rejects shards other than the balanced one, and a missing peer
  ends in DFK_ERR_TIMEOUT at the next sync with the context still usable.
"""
import time

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
TOL = 1e-2


def rel_err(got, ref):
    got = np.asarray(got, dtype=np.float64)
    ref = np.asarray(ref, dtype=np.float64)
    den = np.abs(ref).max()
    return float(np.abs(got - ref).max() / (den if den > 0 else 1.0))


@pytest.fixture(scope="module")
def rt():
    from paper_2602_11808_b200 import runtime
    return runtime


def instance(o, seed, B, dm, df):
    x, wu, wg, wd = o.make_instance(seed, B, dm, df, 1.0 / np.sqrt(dm))
    return tuple(o.quantize_bf16(a)[0] for a in (x, wu, wg, wd))


def chain_ref(o, x0, layers, steps):
    xr = x0
    for _ in range(steps):
        for (wu, wg, wd) in layers:
            xr = o.quantize_bf16(o.forward(xr, wu, wg, wd)[1])[0]
    return xr


def test_graph_recaptured_after_scratch_growth(rt, oracle_lib):
    B, dm, df = 4, 384, 1280
    c = rt.Context(0)
    try:
        layers = [instance(oracle_lib, 900 + l, B, dm, df)[1:] for l in range(2)]
        x0 = instance(oracle_lib, 899, B, dm, df)[0]
        ws = [c.weights(wg, wu, wd) for (wu, wg, wd) in layers]
        xd = c.array((B, dm)).upload(x0)
        yd = c.array((B, dm))
        ref = chain_ref(oracle_lib, x0, layers, 2)
        c.decode(ws, xd, 2, yd, graph=True)
        c.sync()
        assert rel_err(yd.download(), ref) <= 2 * TOL
        # a much larger call grows A2, the down workspace, counters, flags ...
        big = instance(oracle_lib, 898, 200, dm, 4096)
        wb = c.weights(big[2], big[1], big[3])
        xb = c.array((200, dm)).upload(big[0])
        yb = c.array((200, dm), rt.F32)
        c.forward(wb, xb, yb)
        c.sync()
        del wb  # a destroyed weight set also invalidates graphs
        for _ in range(3):  # ... after which the old graph must not be replayed
            yd.fill(0)
            c.decode(ws, xd, 2, yd, graph=True)
            c.sync()
            assert rel_err(yd.download(), ref) <= 2 * TOL
    finally:
        c.close()


def test_graph_over_layers_with_different_tile_counts(rt, oracle_lib):
    B, dm = 3, 256
    dfs = [512, 1536, 640]  # the middle layer has the most stage-1 tiles
    c = rt.Context(0)
    try:
        layers = [instance(oracle_lib, 910 + l, B, dm, df)[1:] for l, df in enumerate(dfs)]
        ws = [c.weights(wg, wu, wd) for (wu, wg, wd) in layers]
        xd = c.array((B, dm))
        yd = c.array((B, dm))
        for rep in range(4):  # new x every replay
            x0 = instance(oracle_lib, 920 + rep, B, dm, 64)[0]
            xd.upload(x0)
            c.decode(ws, xd, 2, yd, graph=True)
            c.sync()
            assert rel_err(yd.download(), chain_ref(oracle_lib, x0, layers, 2)) <= 2 * TOL, rep
    finally:
        c.close()


@pytest.mark.parametrize("B", [9, 12, 16])
def test_gemv_chunks_through_host_async_path(rt, oracle_lib, B):
    dm, df = 384, 1024
    c = rt.Context(0)
    try:
        x, wu, wg, wd = instance(oracle_lib, 930 + B, B, dm, df)
        _, y_ref = oracle_lib.forward(x, wu, wg, wd)
        w = c.weights(wg, wu, wd)
        cfg = rt.Config.make(block_kernel=1, dynamic_sched=1, s1_family=rt.FAMILY_GEMV,
                             down_family=rt.FAMILY_GEMV)
        hx = rt.PinnedHost((B, dm), np.uint16)
        hy = rt.PinnedHost((B, dm), np.float32)
        hx.arr[...] = rt.to_bf16_bits(x)
        for _ in range(3):
            c.forward_host_async(w, hx.arr, hy.arr, cfg=cfg)
        c.sync()
        assert rel_err(hy.arr, y_ref) <= TOL
    finally:
        c.close()


def _ranks(rt, P, dm, max_b):
    ctxs = [rt.Context(0) for _ in range(P)]
    for cx in ctxs:
        cx.tp_sym_create(max_b, dm)
    rt.Context.tp_sym_attach(ctxs)
    return ctxs


@pytest.mark.parametrize("B,fam", [(3, "tc"), (12, "gemv"), (16, "tc")])
def test_fused_tp_writes_y_itself_one_launch(rt, oracle_lib, B, fam):
    P, dm, df = 2, 512, 1601
    x, wu, wg, wd = instance(oracle_lib, 940 + B, B, dm, df)
    _, y_ref = oracle_lib.forward(x, wu, wg, wd)
    cfg = (rt.Config.make(block_kernel=1, dynamic_sched=1, s1_family=rt.FAMILY_GEMV,
                          down_family=rt.FAMILY_GEMV) if fam == "gemv" else None)
    ctxs = _ranks(rt, P, dm, 16)
    try:
        ws = [cx.weights(wg, wu, wd, ff_range=rt.balanced_range(df, P, p))
              for p, cx in enumerate(ctxs)]
        xs = [cx.array((B, dm)).upload(x) for cx in ctxs]
        for dtype in (rt.F32, rt.BF16, rt.F32):
            ys = [cx.array((B, dm), dtype) for cx in ctxs]
            l0 = [cx.launch_count() for cx in ctxs]
            for p, cx in enumerate(ctxs):
                cx.tp_forward_fused(ws[p], xs[p], ys[p], cfg=cfg)
            for cx in ctxs:
                cx.sync()
            chunks = -(-B // 8) if fam == "gemv" else 1
            for p, cx in enumerate(ctxs):
                assert cx.launch_count() - l0[p] == chunks  # no copy / convert after
                assert rel_err(ys[p].download(), y_ref) <= TOL, (dtype, p)
    finally:
        for cx in ctxs:
            cx.close()


def test_fused_tp_rejects_unbalanced_shards(rt, oracle_lib):
    P, dm, df = 2, 256, 256
    x, wu, wg, wd = instance(oracle_lib, 950, 2, dm, df)
    ctxs = _ranks(rt, P, dm, 4)
    try:
        w = ctxs[0].weights(wg, wu, wd, ff_range=(0, 100))  # balanced is (0, 128)
        xd = ctxs[0].array((2, dm)).upload(x)
        yd = ctxs[0].array((2, dm), rt.F32)
        with pytest.raises(rt.InvalidArgument, match="balanced"):
            ctxs[0].tp_forward_fused(w, xd, yd)
    finally:
        for cx in ctxs:
            cx.close()


def test_fused_tp_missing_peer_times_out_recoverably(rt, oracle_lib):
    P, B, dm, df = 2, 2, 256, 512
    x, wu, wg, wd = instance(oracle_lib, 960, B, dm, df)
    _, y_ref = oracle_lib.forward(x, wu, wg, wd)
    ctxs = _ranks(rt, P, dm, 4)
    try:
        ws = [cx.weights(wg, wu, wd, ff_range=rt.balanced_range(df, P, p))
              for p, cx in enumerate(ctxs)]
        xs = [cx.array((B, dm)).upload(x) for cx in ctxs]
        ys = [cx.array((B, dm), rt.F32) for cx in ctxs]
        t0 = time.time()
        ctxs[0].tp_forward_fused(ws[0], xs[0], ys[0])  # rank 1 never joins
        with pytest.raises(rt.TimeoutError_):
            ctxs[0].sync()
        assert time.time() - t0 < 60
        # the context is still usable: fresh symmetric workspaces, both ranks
        for cx in ctxs:
            cx.tp_sym_create(4, dm)
        rt.Context.tp_sym_attach(ctxs)
        for p, cx in enumerate(ctxs):
            cx.tp_forward_fused(ws[p], xs[p], ys[p])
        for cx in ctxs:
            cx.sync()
        for p in range(P):
            assert rel_err(ys[p].download(), y_ref) <= TOL
    finally:
        for cx in ctxs:
            cx.close()


def test_stage_only_weight_sets(rt, oracle_lib):
    """run_fused_stage1 (fused.hpp:61) registers W_up / W_gate alone and
    down_projection (swiglu.hpp:90) W_down alone: each set runs its stage
    and refuses the other (no zero-matrix stand-ins)."""
    B, dm, df = 5, 384, 1000
    x, wu, wg, wd = instance(oracle_lib, 970, B, dm, df)
    a2_ref, y_ref = oracle_lib.forward(x, wu, wg, wd)
    c = rt.Context(0)
    try:
        s1 = c.weights(wg, wu, None)
        dn = c.weights(None, None, wd)
        full = c.weights(wg, wu, wd)
        assert s1.packed_bytes + dn.packed_bytes == full.packed_bytes
        xd = c.array((B, dm)).upload(x)
        a2 = c.array((B, df))
        y = c.array((B, dm), rt.F32)
        for cfg in (None, rt.Config.make(variant=rt.VARIANT_TWO_KERNEL)):
            c.stage1(s1, xd, a2, cfg=cfg)
            c.down(dn, a2, y, cfg=cfg)
            assert rel_err(a2.download(), a2_ref) <= TOL
            assert rel_err(y.download(), y_ref) <= TOL
        with pytest.raises(rt.InvalidArgument):
            c.down(s1, a2, y)
        with pytest.raises(rt.InvalidArgument):
            c.stage1(dn, xd, a2)
        with pytest.raises(rt.InvalidArgument):
            c.forward(s1, xd, y)
    finally:
        c.close()
