"""Host-side plumbing of the tensor-parallel path (one process per GPU).

The GPU work and the all-reduce live in libdfk.so (dfk_tp_init /
dfk_tp_forward, NCCL); this module holds the rank-level logic around it so
it can be exercised on CPU with the gloo backend (tests/test_tp_gloo.py):

* shard_range  — this rank's [ff_begin, ff_end) of d_ff (balanced_ranges,
                 tp.cpp:8-29, through the C ABI);
* exchange_uid — rank 0's 128-byte NCCL unique id broadcast to every rank;
* max_over_ranks — the bench contract's max-over-ranks timing reduction;
* sum_partials — the compound scheme's single all-reduce of partial Y for
                 host-resident fp64 partials (the check the gloo test runs);
* setup_fused  — the fused all-reduce's symmetric workspaces: every rank's
                 64-byte CUDA IPC handle all-gathered, peers opened, and the
                 ranks agree (all or none) on using it.

`dist` is any object with torch.distributed's object collectives
(broadcast_object_list, all_gather_object) -- the launcher's process group;
this module imports no torch itself.
"""
from __future__ import annotations

from typing import Callable, Optional, Tuple

import numpy as np

from . import runtime as rt


def shard_range(d_ff: int, world: int, rank: int) -> Tuple[int, int]:
    return rt.balanced_range(d_ff, world, rank)


def exchange_uid(dist, rank: int, make_uid: Optional[Callable[[], bytes]] = None) -> bytes:
    """Rank 0 creates the NCCL unique id (dfk_tp_unique_id); all ranks get it."""
    box = [None]
    if rank == 0:
        box[0] = (make_uid or rt.Context.tp_unique_id)()
    if dist is not None:
        dist.broadcast_object_list(box, src=0)
    uid = box[0]
    if not isinstance(uid, (bytes, bytearray)) or len(uid) != 128:
        raise ValueError("NCCL unique id must be 128 bytes")
    return bytes(uid)


def _gather(dist, obj) -> list:
    if dist is None:
        return [obj]
    out = [None] * dist.get_world_size()
    dist.all_gather_object(out, obj)
    return out


def max_over_ranks(dist, value: float) -> float:
    return float(max(_gather(dist, float(value))))


def sum_partials(dist, partial: np.ndarray) -> np.ndarray:
    """All-reduce(sum) of a host fp64 partial (one collective of B x d_model),
    summed in rank order like the reference's simulated_all_reduce
    (tp.cpp:90-105)."""
    parts = _gather(dist, np.ascontiguousarray(partial, dtype=np.float64))
    total = np.zeros_like(parts[0])
    for p in parts:
        total += p
    return total


def check_fused(dist, ctx, w, x, y_fused, y_nccl, tol: float = 1e-2) -> Tuple[bool, str]:
    """One call of the fused all-reduce and one of the NCCL comparator on the
    same rank shard and input; every rank must see the same Y within the bf16
    gate and no rank may report a cross-rank timeout.  Returns (all ranks
    ok, this rank's reason) -- the caller falls back to NCCL when not ok, so a
    fused path that misbehaves on a new box never produces the timing."""
    ok, why = 1, "ok"
    try:
        ctx.tp_forward_fused(w, x, y_fused)
        ctx.tp_forward(w, x, y_nccl)
        ctx.sync()
        a = y_fused.download().astype(np.float64)
        b = y_nccl.download().astype(np.float64)
        den = float(np.abs(b).max()) or 1.0
        err = float(np.abs(a - b).max()) / den
        if not np.isfinite(err) or err > tol:
            ok, why = 0, f"fused vs NCCL max rel err {err:.3e} > {tol}"
    except Exception as e:  # noqa: BLE001  (timeout word, CUDA error)
        ok, why = 0, f"{type(e).__name__}: {e}"
    return bool(min(_gather(dist, ok))), why


def setup_fused(dist, ctx, rank: int, world: int, max_batch: int, d_model: int) -> bool:
    """dfk_tp_sym_create on every rank, all-gather the IPC handles,
    dfk_tp_sym_open; True only if every rank succeeded (then all ranks use
    dfk_tp_forward_fused, otherwise all keep the NCCL all-reduce)."""
    ok = 1
    handle = b"\0" * 64
    try:
        handle = ctx.tp_sym_create(max_batch, d_model)
    except Exception:  # noqa: BLE001
        ok = 0
    handles = [handle]
    if dist is not None:
        handles = [None] * world
        dist.all_gather_object(handles, handle)
    if ok:
        try:
            ctx.tp_sym_open(handles, rank, world)
        except Exception:  # noqa: BLE001
            ok = 0
    return bool(min(_gather(dist, ok)))
