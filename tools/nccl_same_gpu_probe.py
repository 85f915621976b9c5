"""Probe: can NCCL build a 2-rank communicator whose ranks share ONE GPU
(two processes, both on cuda:0)?  Prints the dfk_tp_init outcome and, when
it succeeds, runs dfk_tp_forward once per rank against the oracle.

    python -m torch.distributed.run --nproc-per-node 2 --master-addr 127.0.0.1 \
        --master-port 29513 tools/nccl_same_gpu_probe.py
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
ctx = rt.Context(rank % rt.device_count())
box = [rt.Context.tp_unique_id() if rank == 0 else None]
dist.broadcast_object_list(box, src=0)
try:
    ctx.tp_init(box[0], rank, P)
    ok = True
    msg = "ok"
except Exception as e:  # noqa: BLE001
    ok, msg = False, str(e)
print(f"rank {rank}: dfk_tp_init -> {msg}", flush=True)
if ok:
    o = oracle.Oracle()
    B, dm, df = 3, 512, 1537
    x, wu, wg, wd = o.make_instance(7, B, dm, df, 1 / np.sqrt(dm))
    x, wu, wg, wd = (o.quantize_bf16(v)[0] for v in (x, wu, wg, wd))
    _, y_ref = o.forward(x, wu, wg, wd)
    b, e = rt.balanced_range(df, P, rank)
    w = ctx.weights(wg, wu, wd, ff_range=(b, e))
    xd = ctx.array((B, dm)).upload(x)
    yd = ctx.array((B, dm), rt.F32)
    ctx.tp_forward(w, xd, yd)
    ctx.sync()
    y = yd.download().astype(np.float64)
    print(f"rank {rank}: nccl tp_forward rel err "
          f"{np.abs(y - y_ref).max() / np.abs(y_ref).max():.3e}", flush=True)
dist.barrier()
dist.destroy_process_group()
