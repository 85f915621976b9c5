"""World-size-2 CPU test of the tensor-parallel host path (gloo backend).

Each rank takes its balanced_ranges shard of d_ff (through the C ABI), runs
the fp64 oracle on its shard (the GPU kernel's stand-in on a CPU box), and
the ranks combine partial Y with ONE all-reduce — the compound scheme of
tp.cpp:140-167.  Checks: shards partition d_ff, the NCCL-uid exchange and
max-over-ranks reduction work, and the all-reduced Y equals the full-block
oracle and the reference's golden TP output."""
import os
import socket
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out_q):
    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch.distributed as dist
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import oracle
        from paper_2602_11808_b200 import tp_host
        o = oracle.Oracle()
        o.threads = 1
        golden = np.load(os.path.join(ROOT, "tests", "golden", "golden.npz"))
        seed, B, dm, df, _ = (int(v) for v in golden["tp_3x6x12/meta"])
        x, wu, wg, wd = o.make_instance(seed, B, dm, df, 1.0)
        b, e = tp_host.shard_range(df, world, rank)
        uid = tp_host.exchange_uid(dist, rank, make_uid=lambda: bytes(range(128)))
        _, yp = o.forward(x, np.ascontiguousarray(wu[:, b:e]),
                          np.ascontiguousarray(wg[:, b:e]),
                          np.ascontiguousarray(wd[b:e, :]))
        y = tp_host.sum_partials(dist, yp)
        t = tp_host.max_over_ranks(dist, float(rank + 1))
        _, y_full = o.forward(x, wu, wg, wd)
        out_q.put((rank, (b, e), uid == bytes(range(128)), t,
                   float(np.abs(y - y_full).max()),
                   float(np.abs(y - golden[f"tp_3x6x12/tp{world}"]).max())))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_tp_world2_gloo(world):
    import multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=180) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    ranges = [r[1] for r in res]
    assert ranges[0][0] == 0 and ranges[-1][1] == 12
    assert all(ranges[i][1] == ranges[i + 1][0] for i in range(world - 1))
    for rank, _, uid_ok, tmax, err_full, err_golden in res:
        assert uid_ok
        assert tmax == float(world)          # max over ranks
        assert err_full <= 1e-12 and err_golden <= 1e-12
