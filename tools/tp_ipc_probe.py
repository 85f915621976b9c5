"""Multi-process check of the fused TP all-reduce's IPC path: N processes
(torch.distributed gloo for the handle exchange only), each maps its peers'
symmetric workspaces with cudaIpcOpenMemHandle and runs dfk_tp_forward_fused
on its balanced_ranges shard; rank 0 compares every rank's Y with the
oracle.  With one GPU visible all ranks share cuda:0 (the GPU time-slices
between the processes' contexts, so this checks the protocol, not speed).

    python -m torch.distributed.run --nproc-per-node 2 --master-addr 127.0.0.1 \
        --master-port 29511 tools/tp_ipc_probe.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch.distributed as dist  # noqa: E402

import oracle  # noqa: E402
from paper_2602_11808_b200 import runtime as rt  # noqa: E402

dist.init_process_group("gloo")
rank, P = dist.get_rank(), dist.get_world_size()
ndev = rt.device_count() if hasattr(rt, "device_count") else 1
ctx = rt.Context(rank % max(1, ndev))
o = oracle.Oracle()
B, dm, df = 3, 512, 1537
x, wu, wg, wd = o.make_instance(7, B, dm, df, 1 / np.sqrt(dm))
x, wu, wg, wd = (o.quantize_bf16(v)[0] for v in (x, wu, wg, wd))
_, y_ref = o.forward(x, wu, wg, wd)
h = ctx.tp_sym_create(16, dm)
hs = [None] * P
dist.all_gather_object(hs, h)
ctx.tp_sym_open(hs, rank, P)
b, e = rt.balanced_range(df, P, rank)
w = ctx.weights(wg, wu, wd, ff_range=(b, e))
xd = ctx.array((B, dm)).upload(x)
yd = ctx.array((B, dm), rt.F32)
errs = []
for rep in range(3):
    dist.barrier()
    ctx.tp_forward_fused(w, xd, yd)
    ctx.sync()
    y = yd.download().astype(np.float64)
    errs.append(float(np.abs(y - y_ref).max() / np.abs(y_ref).max()))
allerr = [None] * P
dist.all_gather_object(allerr, errs)
if rank == 0:
    worst = max(max(v) for v in allerr)
    print(f"tp ipc probe P={P}: max rel err over ranks/reps {worst:.3e}",
          "OK" if worst <= 1e-2 else "FAIL", flush=True)
dist.barrier()
ctx.close()
dist.destroy_process_group()
