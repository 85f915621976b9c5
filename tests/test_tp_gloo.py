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


class _FakeSymCtx:
    """Stands in for a Context on a CPU box: records the IPC-handle exchange
    of tp_host.setup_fused; `fail_open` makes this rank's peer mapping fail."""

    def __init__(self, rank, fail_open):
        self.rank, self.fail_open, self.opened = rank, fail_open, None

    def tp_sym_create(self, max_batch, d_model):
        return bytes([self.rank]) * 64

    def tp_sym_open(self, handles, rank, world):
        if self.fail_open:
            raise RuntimeError("cudaIpcOpenMemHandle failed")
        self.opened = list(handles)


def _sym_worker(rank, world, port, fail_rank, out_q):
    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch.distributed as dist
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2602_11808_b200 import tp_host
        c = _FakeSymCtx(rank, rank == fail_rank)
        ok = tp_host.setup_fused(dist, c, rank, world, 64, 4096)
        out_q.put((rank, ok, c.opened))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("fail_rank", [-1, 1])
def test_fused_tp_handle_exchange_gloo(fail_rank):
    """setup_fused: every rank receives every rank's 64-byte handle in rank
    order, and the ranks agree -- one rank failing to map its peers makes ALL
    ranks keep the NCCL all-reduce (a split decision would deadlock)."""
    import multiprocessing as mp
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_sym_worker, args=(r, world, port, fail_rank, q))
             for r in range(world)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=180) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, ok, opened in res:
        assert ok == (fail_rank < 0)
        if rank != fail_rank:
            assert opened == [bytes([r]) * 64 for r in range(world)]


class _FakeArr:
    def __init__(self, v):
        self.v = np.asarray(v, dtype=np.float32)

    def download(self):
        return self.v


class _FakeCtx:
    """Stands in for a rank's context: the fused and the NCCL all-reduce
    write given Y values (or the fused one raises, like a cross-rank
    timeout reported by dfk_context_sync)."""

    def __init__(self, fused, nccl, raise_fused=False):
        self.fused, self.nccl, self.raise_fused = fused, nccl, raise_fused

    def tp_forward_fused(self, w, x, y):
        if self.raise_fused:
            raise RuntimeError("[dfk status 9] peer rank timed out")
        y.v[...] = self.fused

    def tp_forward(self, w, x, y):
        y.v[...] = self.nccl

    def sync(self):
        pass


def _check_worker(rank, world, port, case, out_q):
    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch.distributed as dist
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2602_11808_b200 import tp_host
        good = np.linspace(-1.0, 1.0, 8)
        bad = good + (0.5 if (case == "mismatch" and rank == 1) else 0.0)
        ctx = _FakeCtx(bad, good, raise_fused=(case == "timeout" and rank == 0))
        ok, why = tp_host.check_fused(dist, ctx, None, None, _FakeArr(np.zeros(8)),
                                      _FakeArr(np.zeros(8)))
        out_q.put((rank, ok, why))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("case,want", [("agree", True), ("mismatch", False), ("timeout", False)])
def test_fused_allreduce_self_check_all_ranks_agree(case, want):
    """bench.py's first-contact check of the fused all-reduce (tp_host.check_fused):
    one rank's disagreement with NCCL or a timeout makes EVERY rank fall back."""
    import multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_check_worker, args=(r, 2, port, case, q)) for r in range(2)]
    for p in ps:
        p.start()
    res = sorted(q.get(timeout=120) for _ in ps)
    for p in ps:
        p.join(timeout=60)
    assert [r[1] for r in res] == [want, want], res
    if case == "mismatch":
        assert "max rel err" in res[1][2]
    if case == "timeout":
        assert "timed out" in res[0][2]
