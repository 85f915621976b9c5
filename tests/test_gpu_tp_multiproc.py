"""Tensor parallelism across PROCESSES (one process per rank, the reference's
compound scheme tp.cpp:140-167 with its one all-reduce):

* the fused all-reduce (dfk_tp_forward_fused) with the ranks' symmetric
  workspaces mapped through CUDA IPC handles (dfk_tp_sym_create / _open) --
  with one visible GPU both processes share it (time-sliced contexts: this
  checks the cross-process protocol, not speed); with >= 2 GPUs each rank
  has its own device and the partial sums cross NVLink;
* the NCCL comparator (dfk_tp_init + dfk_tp_forward), which needs one GPU per
  rank (NCCL rejects two ranks on one device), so it runs only when >= 2 GPUs
  are visible.

Every rank's Y is checked against the fp64 oracle on the same bf16 inputs
(tolerance of the north star, max|dY|/max|Y| <= 1e-2)."""
import multiprocessing as mp

import pytest

import dfk_tp_ranks as _tp_worker

pytestmark = pytest.mark.gpu
TOL = 1e-2


def _gpus():
    from paper_2602_11808_b200 import runtime as rt
    return rt.device_count()


def _run(target, P, args_for, relay, timeout=240):
    ctx = mp.get_context("spawn")
    pipes = [ctx.Pipe() for _ in range(P)]
    procs = [ctx.Process(target=target, args=(r, P, pipes[r][1], *args_for(r)))
             for r in range(P)]
    for p in procs:
        p.start()
    try:
        results = relay([pp[0] for pp in pipes], timeout)
    finally:
        for p in procs:
            p.join(timeout=60)
            if p.is_alive():
                p.kill()
    return results


def _recv(conn, timeout):
    if not conn.poll(timeout):
        raise TimeoutError("rank did not answer")
    kind, payload = conn.recv()
    if kind == "error":
        raise AssertionError(f"rank failed: {payload}")
    return kind, payload


@pytest.mark.parametrize("P,B,df", [(2, 3, 1537), (2, 12, 1024), (3, 5, 1100)])
def test_fused_allreduce_across_processes(P, B, df):
    dm = 512
    ngpu = _gpus()

    def relay(conns, timeout):
        handles = [_recv(c, timeout)[1] for c in conns]
        for c in conns:
            c.send(handles)
        return [_recv(c, timeout)[1] for c in conns]

    res = _run(_tp_worker.fused_rank, P,
               lambda r: (r % ngpu, B, dm, df, 41 + P + B), relay)
    for r, out in enumerate(res):
        assert max(out["errs"]) <= TOL, (r, out)
        # the all-reduce lives in the block kernel: one launch per block
        assert out["launches_per_block"] == 1, (r, out)


@pytest.mark.skipif("_gpus() < 2", reason="NCCL needs one GPU per rank (>= 2 visible)")
def test_nccl_allreduce_across_processes():
    P = min(_gpus(), 4)
    B, dm, df = 4, 512, 1537

    def relay(conns, timeout):
        uid = _recv(conns[0], timeout)[1]
        for c in conns:
            c.send(uid)
        return [_recv(c, timeout)[1] for c in conns]

    res = _run(_tp_worker.nccl_rank, P, lambda r: (B, dm, df, 77), relay)
    for r, out in enumerate(res):
        assert max(out["errs"]) <= TOL, (r, out)
