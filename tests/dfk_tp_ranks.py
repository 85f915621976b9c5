"""Worker processes of the multi-process tensor-parallel tests (one process
per rank, the way a serving stack runs the path).  The parent hands out the
rank and pipes; handles / NCCL ids are exchanged through the parent, so no
torch.distributed is involved (tests/test_gpu_tp_multiproc.py)."""
import numpy as np


def _instance(seed, B, dm, df):
    import oracle
    o = oracle.Oracle()
    x, wu, wg, wd = o.make_instance(seed, B, dm, df, 1.0 / np.sqrt(dm))
    return o, tuple(o.quantize_bf16(a)[0] for a in (x, wu, wg, wd))


def _rel(got, ref):
    got = np.asarray(got, np.float64)
    ref = np.asarray(ref, np.float64)
    return float(np.abs(got - ref).max() / max(np.abs(ref).max(), 1e-30))


def fused_rank(rank, P, conn, device, B, dm, df, seed):
    """dfk_tp_sym_create -> 64-byte CUDA IPC handle to the parent -> every
    rank's handle back -> dfk_tp_sym_open -> fp32 and bf16 fused-TP blocks
    and a 2-layer decode chain, each checked against the oracle."""
    try:
        from paper_2602_11808_b200 import runtime as rt
        o, (x, wu, wg, wd) = _instance(seed, B, dm, df)
        _, y_ref = o.forward(x, wu, wg, wd)
        ctx = rt.Context(device)
        conn.send(("handle", ctx.tp_sym_create(max(B, 8), dm)))
        handles = conn.recv()
        ctx.tp_sym_open(handles, rank, P)
        b, e = rt.balanced_range(df, P, rank)
        w = ctx.weights(wg, wu, wd, ff_range=(b, e))
        xd = ctx.array((B, dm)).upload(x)
        out = {}
        errs = []
        y32 = ctx.array((B, dm), rt.F32)
        l0 = ctx.launch_count()
        for _ in range(3):
            ctx.tp_forward_fused(w, xd, y32)
        ctx.sync()
        out["launches_per_block"] = (ctx.launch_count() - l0) / 3
        errs.append(_rel(y32.download(), y_ref))
        y16 = ctx.array((B, dm))
        ctx.tp_forward_fused(w, xd, y16)
        ctx.sync()
        errs.append(_rel(y16.download(), y_ref))
        # decode chain: 2 layers x 2 steps, eager then graph-replayed twice
        layers = [_instance(seed + 1 + l, B, dm, df)[1][1:] for l in range(2)]
        xr = x
        for _ in range(2):
            for (lu, lg, ld) in layers:
                xr = o.quantize_bf16(o.forward(xr, lu, lg, ld)[1])[0]
        ws = [ctx.weights(lg, lu, ld, ff_range=(b, e)) for (lu, lg, ld) in layers]
        yd = ctx.array((B, dm))
        for graph in (False, True, True):
            ctx.decode(ws, xd, 2, yd, graph=graph)
            ctx.sync()
            errs.append(_rel(yd.download(), xr) / 2)  # chain tolerance is 2x
        out["errs"] = errs
        conn.send(("ok", out))
        ctx.close()
    except Exception as e:  # noqa: BLE001
        conn.send(("error", repr(e)))


def nccl_rank(rank, P, conn, B, dm, df, seed):
    """dfk_tp_init over a parent-relayed ncclUniqueId, then dfk_tp_forward
    (block -> fp32 partial -> one ncclAllReduce) on this rank's GPU."""
    try:
        from paper_2602_11808_b200 import runtime as rt
        o, (x, wu, wg, wd) = _instance(seed, B, dm, df)
        _, y_ref = o.forward(x, wu, wg, wd)
        ctx = rt.Context(rank)
        if rank == 0:
            conn.send(("uid", rt.Context.tp_unique_id()))
        uid = conn.recv()
        ctx.tp_init(uid, rank, P)
        b, e = rt.balanced_range(df, P, rank)
        w = ctx.weights(wg, wu, wd, ff_range=(b, e))
        xd = ctx.array((B, dm)).upload(x)
        y = ctx.array((B, dm), rt.F32)
        errs = []
        for _ in range(3):
            ctx.tp_forward(w, xd, y)
            ctx.sync()
            errs.append(_rel(y.download(), y_ref))
        conn.send(("ok", {"errs": errs}))
        ctx.close()
    except Exception as e:  # noqa: BLE001
        conn.send(("error", repr(e)))
