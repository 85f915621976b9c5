#!/usr/bin/env python
"""Benchmark of the fused SwiGLU-MLP decode path (BASELINE.json metric:
"SwiGLU-MLP decode µs/call & achieved HBM GB/s vs ~8 TB/s roofline, batch
1-64").

Workload (configs[1]): Llama-3.1-8B MLP (d_model=4096, d_ff=14336), batch
sweep B in {1,2,4,8,16,32,64} on one B200, scheduler-selected kernels.  A
"step" is one fused block call at every B of the sweep (7 calls), each on the
next of R rotating weight sets (every set is 352 MB >> 126 MB L2, so no call
finds its weights in L2).  Synthetic bf16 data (uniform, device-generated).

value      = algorithmic bytes of all calls / device time (GB/s, aggregate
             over ranks); bytes per call follow the reference's fused traffic
             model (traffic.cpp:70-76, 82-94) at 2 B/element.
e2e        = the same metric through the host-buffer C-ABI call
             (dfk_forward_host_async: X bf16 from pinned host memory, H2D on a
             side stream gated by device flags, Y fp32 D2H on a second side
             stream once the block's last CTA flags it; one host sync per
             step, which waits for every copy).
roofline   = the fused stage-1 kernel (2/3 of the bytes) timed alone with
             CUDA events on its stream, against MEASURED_PEAKS.json hbm_gbs.
cpu_baseline = the reference CPU path (oracle/_ref, the unmodified reference
             compiled in place) on a bounded sample.

N>1 (torchrun): tensor parallel over NCCL, one rank per GPU — every rank holds
the balanced_ranges(d_ff, N) shard and the block ends in one ncclAllReduce.

Extra keys: decode_loop (configs[2]: Qwen2.5-7B, 4-layer x<-Y decode loop,
CUDA graph) and tp_rank_blocks (configs[3]/[4]: the per-rank block of the
Qwen2.5-32B / Llama-3.1-70B tensor-parallel shards, on this one GPU).

--impl reference: the reference's own CPU implementation of the path
(oracle/_ref/libdeepfusion_ref.so: run_fused with a single covering
column-major tile and all host threads) on rank 0, same metric/unit.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

DM, DF = 4096, 14336
SWEEP = [1, 2, 4, 8, 16, 32, 64]
METRIC = "SwiGLU-MLP decode µs/call & achieved HBM GB/s vs ~8 TB/s roofline, batch 1–64"
WORKLOAD = "Llama-3.1-8B MLP (d_model=4096, d_ff=14336) decode batch sweep 1/2/4/8/16/32/64"


def block_bytes(B, dm, df, P=1):
    """Per-GPU algorithmic bytes of one block call at TP degree P."""
    return 2 * (3 * dm * df // P + 2 * B * dm + 2 * B * df // P)


def stream_floor():
    """The bare cp.async.bulk stream of one Llama-8B block's bytes per launch,
    PDL-chained, on this GPU (tools/stream_probe launch): the best a single
    launch of this size streams -- context for roofline.frac, whose peak is
    MEASURED_PEAKS.json's copy bandwidth."""
    exe = os.path.join(ROOT, "tools", "stream_probe")
    if not os.path.exists(exe):
        return None
    try:
        out = subprocess.run([exe, "launch"], capture_output=True, text=True,
                             timeout=60).stdout
    except Exception:  # noqa: BLE001
        return None
    best = None
    for ln in out.splitlines():
        if ln.startswith("launch") and "pdl=1" in ln and "GB/s" in ln:
            us = float(ln.split(":")[1].split("us/launch")[0])
            gbs = float(ln.split("us/launch")[1].split("GB/s")[0])
            if best is None or gbs > best["gbs"]:
                best = {"us_per_352MB_launch": us, "gbs": gbs,
                        "how": "tools/stream_probe launch: bare cp.async.bulk ring, "
                               "352 MB per launch, PDL-chained, best grid/chunk"}
    return best


def measured_peak():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


# --- clocks sampling ---------------------------------------------------------
class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "50"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except FileNotFoundError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        if self.proc:
            time.sleep(0.25)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for n, v in zip(names, parts[3:7]):
                if v.lower() == "active":
                    reasons.add(n)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(mx),
                "reasons": sorted(reasons), "samples": len(sm)}


# --- reference CPU arm -------------------------------------------------------
class CpuReference:
    """The reference CPU path (oracle/_ref: the unmodified reference compiled
    in place) on a Llama-8B-shaped fp64 instance built once."""

    def __init__(self, B=1):
        import oracle
        o = oracle.Oracle()
        self.B = B
        x, wu, wg, wd = o.make_instance(0, B, DM, DF, 1.0 / np.sqrt(DM))
        self.inst = oracle.Reference().instance(x, wu, wg, wd)

    def time(self, threads=1, budget_s=12.0, min_calls=3, max_calls=50):
        """run_fused (fused.cpp:209-216, single covering column-major tile,
        `threads` stage-1 workers); returns (GB/s of algorithmic bytes,
        calls, median seconds per call)."""
        tile = (self.B, -(-DF // threads) if threads > 1 else DF, DM)
        self.inst.run_fused(tile=tile, num_workers=threads)  # warm-up
        times = []
        t_start = time.perf_counter()
        while len(times) < max_calls and (len(times) < min_calls or
                                          time.perf_counter() - t_start < budget_s):
            t0 = time.perf_counter()
            self.inst.run_fused(tile=tile, num_workers=threads)
            times.append(time.perf_counter() - t0)
        per_call = statistics.median(times)
        return block_bytes(self.B, DM, DF) / per_call / 1e9, len(times), per_call


def _cpu_model():
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    return None


def run_reference_arm(args, rank, world):
    if rank != 0:
        return
    threads = os.cpu_count() or 1
    t_all = time.perf_counter()
    ref = CpuReference(B=1)
    vals = []
    for step in range(args.warmup + args.steps):
        gbs, n, per = ref.time(threads=threads, budget_s=0.0, min_calls=1, max_calls=1)
        if step >= args.warmup:
            vals.append((gbs, per))
    gbs = statistics.median(v[0] for v in vals)
    per = statistics.median(v[1] for v in vals)
    line = {
        "impl": "reference", "metric": METRIC, "value": round(gbs, 4), "unit": "GB/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(per * 1e3, 3), "higher_is_better": True,
        "scaling": "strong" if args.gpus > 1 else "weak", "vs_baseline": None,
        "dtype": "f64", "data": "synthetic (mt19937_64 uniform, reference generator)",
        "config": {"workload": WORKLOAD, "sample": "one B=1 block per step",
                   "parallelism": f"{threads} host threads (stage 1), down single-thread"},
        "cpu_baseline": {"value": round(gbs, 4), "unit": "GB/s", "cores": threads,
                         "kind": "reference", "cpu_model": _cpu_model(),
                         "sample": f"reference run_fused, Llama-8B B=1, {threads} stage-1 "
                                   f"workers, one call per step"},
        "e2e": {"value": round(gbs, 4), "unit": "GB/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
        "us_per_call": {"1": round(per * 1e6, 1)},
        "wall_s": round(time.perf_counter() - t_all, 1),
    }
    print(json.dumps(line), flush=True)


# --- config 3: Qwen2.5-7B multi-layer decode loop -----------------------------
QWEN7_DM, QWEN7_DF = 3584, 18944


def decode_loop(rt, ctx, ev0, ev1, layers=4, steps=8, sweep=(1, 2, 4, 8, 16, 32)):
    """BASELINE configs[2]: Qwen2.5-7B MLP, `layers` distinct layers (4 x 407 MB
    >> L2), `steps` decode steps with x <- Y (bf16) after every block
    (time_decode_seconds, bench.cpp:98-115), the whole sequence captured once
    into a CUDA graph (dfk_decode) and replayed; tokens/s = B * steps / s."""
    dm, df = QWEN7_DM, QWEN7_DF
    scale = 1.0 / np.sqrt(dm)
    ws = []
    for l in range(layers):
        g = ctx.array((dm, df)).fill_uniform(5000 + 3 * l, -scale, scale)
        u = ctx.array((dm, df)).fill_uniform(5001 + 3 * l, -scale, scale)
        d = ctx.array((df, dm)).fill_uniform(5002 + 3 * l, -scale, scale)
        ws.append(ctx.weights(g, u, d))
        del g, u, d
    out = {"model": "Qwen2.5-7B MLP (d_model=3584, d_ff=18944)", "layers": layers,
           "steps": steps, "graph": True, "per_batch": {}}
    for B in sweep:
        x = ctx.array((B, dm)).fill_uniform(77 + B)
        y = ctx.array((B, dm))
        res = {}
        for graph in (True, False):
            for _ in range(2):
                ctx.decode(ws, x, steps, y, graph=graph)
            ctx.sync()
            # 4 timed repetitions, mean +- population std of tokens/s
            # (bench.cpp:59-67 compute_stats, "measured four times")
            times = []
            for _ in range(4):
                ev0.record(ctx)
                ctx.decode(ws, x, steps, y, graph=graph)
                ev1.record(ctx)
                ctx.sync()
                times.append(ev0.elapsed_ms(ev1) * 1e-3)
            res[graph] = times
        t = statistics.mean(res[True])
        tps = [B * steps / v for v in res[True]]
        blocks = layers * steps
        out["per_batch"][str(B)] = {
            "tokens_per_s": round(statistics.mean(tps), 1),
            "tokens_per_s_std": round(statistics.pstdev(tps), 1),
            "us_per_block": round(t / blocks * 1e6, 2),
            "gbs": round(block_bytes(B, dm, df) * blocks / t / 1e9, 1),
            "eager_us_per_block": round(statistics.mean(res[False]) / blocks * 1e6, 2),
        }
    del ws
    return out


# --- configs 4/5: the per-rank block of the tensor-parallel configs ------------
TP_SHAPES = (("Qwen2.5-32B", 5120, 27648, (1, 2, 4, 8)),
             ("Llama-3.1-70B", 8192, 28672, (2, 4, 8)))


def tp_shards(rt, ctx, ev0, ev1, batches=(1, 16, 64), reps=20, tune=True):
    """BASELINE configs[3] / [4] on ONE GPU: a rank of TP=P runs the block of
    its balanced_ranges(d_ff, P) shard (tp.cpp:8-29), so its kernel time is
    that block's time (the all-reduce, fused in the kernel at N > 1, is not in
    this number).  `us`: the library default config (what a NULL-config call
    runs); `tuned_us`: the scheduler's pick for that shard and batch (dfk_tune,
    tuner.cpp's profile/select).  Weight sets rotated beyond 3x L2."""
    import math
    out = {}
    for name, dm, df, Ps in TP_SHAPES:
        for P in Ps:
            b0, b1 = rt.balanced_range(df, P, 0)
            dfs = b1 - b0
            nsets = max(2, math.ceil(3 * 126e6 / (3 * dm * dfs * 2)))
            s = 1.0 / np.sqrt(dm)
            ws = []
            for i in range(nsets):
                g = ctx.array((dm, dfs)).fill_uniform(9000 + 3 * i, -s, s)
                u = ctx.array((dm, dfs)).fill_uniform(9001 + 3 * i, -s, s)
                d = ctx.array((dfs, dm)).fill_uniform(9002 + 3 * i, -s, s)
                ws.append(ctx.weights(g, u, d))
                del g, u, d
            row = {}
            for B in batches:
                x = ctx.array((B, dm)).fill_uniform(31 + B)
                y = ctx.array((B, dm), rt.F32)

                def run(cfg):
                    for i in range(4):
                        ctx.forward(ws[i % nsets], x, y, cfg=cfg)
                    ctx.sync()
                    ev0.record(ctx)
                    for i in range(reps):
                        ctx.forward(ws[i % nsets], x, y, cfg=cfg)
                    ev1.record(ctx)
                    ctx.sync()
                    return ev0.elapsed_ms(ev1) * 1e3 / reps

                if tune:
                    # tune first, then time default and pick alternately (the
                    # tuning burst can leave the GPU at its power cap for a while)
                    # (after dfk_tune a NULL config runs the pick: keep the
                    # library default's resolved config)
                    dcfg = ctx.resolve_config(ws[0], B)
                    cfg, _, _ = ctx.tune(ws[0], B, None, 1, 4)
                    time.sleep(1.0)  # let the power controller settle after the burst
                    t = [run(dcfg), run(cfg), run(dcfg), run(cfg)]
                    us, tus = (t[0] + t[2]) / 2, (t[1] + t[3]) / 2
                else:
                    us = run(None)
                gbs = block_bytes(B, dm, dfs) / (us * 1e-6) / 1e9
                row[str(B)] = {"us": round(us, 2), "gbs": round(gbs, 1)}
                if tune:
                    row[str(B)].update({
                        "tuned_us": round(tus, 2),
                        "tuned_gbs": round(block_bytes(B, dm, dfs) / (tus * 1e-6) / 1e9, 1),
                        "tuned_cfg": cfg.label.decode()})
            out[f"{name} tp{P}"] = {"d_model": dm, "d_ff_shard": dfs, "per_batch": row}
            del ws
    return out


# --- configs 4/5 at N > 1: the whole tensor-parallel block, all-reduce included
def tp_configs(rt, ctx, ev0, ev1, rank, P, tp_mode, barrier, max_over_ranks,
               batches=(1, 16, 64), reps=20):
    """BASELINE configs[3] (Qwen2.5-32B, TP 1/2/4/8) and configs[4]
    (Llama-3.1-70B, TP 2/4/8) end to end on P ranks: every rank holds its
    balanced_ranges shard (tp.cpp:8-29), the block ends in the ONE
    all-reduce (tp.cpp:140-167) -- fused into the block kernel over NVLink
    peer memory when tp_mode is "fused-nvlink", and NCCL's ncclAllReduce
    after the block as the comparator.  µs per call = max over ranks of the
    event-timed mean over `reps` calls on rotating weight sets (> 3x L2)."""
    import math
    out = {}
    for name, dm, df, Ps in TP_SHAPES:
        if P not in Ps:
            continue
        b0, b1 = rt.balanced_range(df, P, rank)
        dfs = b1 - b0
        nsets = max(2, math.ceil(3 * 126e6 / (3 * dm * dfs * 2)))
        s = 1.0 / np.sqrt(dm)
        ws = []
        for i in range(nsets):
            g = ctx.array((dm, df)).fill_uniform(9000 + 3 * i, -s, s)
            u = ctx.array((dm, df)).fill_uniform(9001 + 3 * i, -s, s)
            d = ctx.array((df, dm)).fill_uniform(9002 + 3 * i, -s, s)
            ws.append(ctx.weights(g, u, d, ff_range=(b0, b1)))
            del g, u, d
        ctx.sync()
        row = {}
        for B in batches:
            x = ctx.array((B, dm)).fill_uniform(31 + B)
            y = ctx.array((B, dm), rt.F32)
            arms = {}
            fns = {"nccl": lambda w: ctx.tp_forward(w, x, y)}
            if tp_mode == "fused-nvlink":
                fns["fused"] = lambda w: ctx.tp_forward_fused(w, x, y)
            for arm, fn in fns.items():
                for i in range(4):
                    fn(ws[i % nsets])
                ctx.sync()
                barrier()
                ev0.record(ctx)
                for i in range(reps):
                    fn(ws[i % nsets])
                ev1.record(ctx)
                ctx.sync()
                arms[arm] = max_over_ranks(ev0.elapsed_ms(ev1) * 1e3 / reps)
            us = arms.get("fused", arms["nccl"])
            gbs = block_bytes(B, dm, df // P) * P / (us * 1e-6) / 1e9
            row[str(B)] = {"us": round(us, 2), "gbs_aggregate": round(gbs, 1),
                           "nccl_allreduce_us": round(arms["nccl"], 2)}
        out[f"{name} tp{P}"] = {"d_model": dm, "d_ff": df, "d_ff_shard": dfs,
                                "allreduce": tp_mode, "per_batch": row}
        del ws
    return out


# --- launcher: `bench.py --gpus N` without torchrun ----------------------------
def self_launch(args) -> int:
    """Starts N ranks of this script (one process per GPU, RANK / LOCAL_RANK /
    WORLD_SIZE / MASTER_* in the environment, rendezvous on 127.0.0.1), the
    way torchrun would; fails if fewer than N GPUs are visible."""
    import socket
    try:
        out = subprocess.run(["nvidia-smi", "-L"], capture_output=True, text=True,
                             timeout=60).stdout
        visible = sum(1 for ln in out.splitlines() if ln.startswith("GPU "))
    except Exception:  # noqa: BLE001
        visible = 0
    cvd = os.environ.get("CUDA_VISIBLE_DEVICES")
    if cvd is not None:
        visible = min(visible, len([d for d in cvd.split(",") if d.strip()]))
    if visible < args.gpus and not args.tp_emulate:
        print(f"bench.py: --gpus {args.gpus} needs {args.gpus} visible GPUs, "
              f"found {visible}", file=sys.stderr, flush=True)
        return 1
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    procs = []
    for r in range(args.gpus):
        env = dict(os.environ, RANK=str(r), LOCAL_RANK=str(r), WORLD_SIZE=str(args.gpus),
                   LOCAL_WORLD_SIZE=str(args.gpus), MASTER_ADDR="127.0.0.1",
                   MASTER_PORT=str(port))
        env.setdefault("NCCL_DEBUG", "INFO")
        procs.append(subprocess.Popen([sys.executable, os.path.abspath(__file__)] + sys.argv[1:],
                                      env=env))
    rc = 0
    for p in procs:
        rc = max(rc, p.wait())
    return rc


# --- GPU arm -----------------------------------------------------------------
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--sets", type=int, default=4, help="rotating weight sets")
    ap.add_argument("--no-tune", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-decode", action="store_true")
    ap.add_argument("--no-tp-shards", action="store_true")
    ap.add_argument("--tp-emulate", action="store_true",
                    help="test aid: ranks share the visible GPUs (rank %% count), no NCCL")
    ap.add_argument("--sweep", default=",".join(map(str, SWEEP)))
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    sweep = [int(b) for b in args.sweep.split(",")]

    if (args.gpus > 1 and "WORLD_SIZE" not in os.environ and args.impl == "ours"):
        sys.exit(self_launch(args))
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if args.impl == "ours" and world != args.gpus:
        print(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}", file=sys.stderr)
        sys.exit(1)
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    dist = None
    if world > 1:
        import torch.distributed as dist  # plumbing only: rendezvous + max-reduce
        dist.init_process_group("gloo")
    if args.impl == "reference":
        run_reference_arm(args, rank, world)
        if dist:
            dist.barrier()
            dist.destroy_process_group()
        return

    from paper_2602_11808_b200 import runtime as rt
    from paper_2602_11808_b200 import tp_host

    P = world
    if not args.tp_emulate and local_rank >= rt.device_count():
        raise SystemExit(f"bench.py: rank {rank} needs GPU {local_rank}, "
                         f"{rt.device_count()} visible")
    dev = local_rank % rt.device_count() if args.tp_emulate else local_rank
    ctx = rt.Context(dev)
    tp_mode = None
    if P > 1:
        # NCCL (the unfused-collective comparator) and the fused all-reduce's
        # symmetric workspaces over NVLink peer memory (used when every rank
        # can map its peers).
        if not args.tp_emulate:
            ctx.tp_init(tp_host.exchange_uid(dist, rank), rank, P)
        sweep_max = max(int(b) for b in args.sweep.split(","))
        tp_mode = ("fused-nvlink" if tp_host.setup_fused(dist, ctx, rank, P, sweep_max, DM)
                   else "nccl")
    f0, f1 = tp_host.shard_range(DF, P, rank)

    def barrier():
        if dist:
            dist.barrier()

    def max_over_ranks(v):
        return tp_host.max_over_ranks(dist, v)

    # Weight sets: synthetic bf16 U[-1/sqrt(dm), 1/sqrt(dm)) generated on the
    # device in the reference layout, then prepacked (sources freed).
    scale = 1.0 / np.sqrt(DM)
    sets = []
    for s in range(args.sets):
        g = ctx.array((DM, DF)).fill_uniform(1000 * s + 1, -scale, scale)
        u = ctx.array((DM, DF)).fill_uniform(1000 * s + 2, -scale, scale)
        d = ctx.array((DF, DM)).fill_uniform(1000 * s + 3, -scale, scale)
        sets.append(ctx.weights(g, u, d, ff_range=(f0, f1)))
        del g, u, d
    ctx.sync()
    bmax = max(sweep)
    xs = {B: ctx.array((B, DM)).fill_uniform(7 + B) for B in sweep}
    ys = {B: ctx.array((B, DM), rt.F32) for B in sweep}
    fused_check = None
    if tp_mode == "fused-nvlink" and not args.tp_emulate:
        # first contact with a multi-GPU box: the fused all-reduce must agree
        # with NCCL (and not time out) on every rank before it is timed
        yn = ctx.array((bmax, DM), rt.F32)
        ok, why = tp_host.check_fused(dist, ctx, sets[0], xs[bmax], ys[bmax], yn)
        fused_check = "ok" if ok else f"fell back to NCCL ({why} on rank {rank})"
        if not ok:
            tp_mode = "nccl"
        del yn

    # Scheduler: profile once per batch size (tuner.cpp get_or_tune).
    chosen = {}
    if not args.no_tune:
        for B in sweep:
            cfg, hit, entry = ctx.tune(sets[0], B, None, 1, 4)
            chosen[B] = cfg.label.decode()
        time.sleep(1.0)  # let the power controller settle after the tuning burst
    cfgs = {B: ctx.select_config(sets[0], B) for B in sweep}

    def call(B, i, cfg=None):
        w = sets[i % len(sets)]
        if tp_mode == "fused-nvlink":
            ctx.tp_forward_fused(w, xs[B], ys[B], cfg=cfg)
        elif P > 1:
            ctx.tp_forward(w, xs[B], ys[B], cfg=cfg)
        else:
            ctx.forward(w, xs[B], ys[B], cfg=cfg)

    def nccl_call(B, i, cfg=None):
        ctx.tp_forward(sets[i % len(sets)], xs[B], ys[B], cfg=cfg)

    def step(k):
        for j, B in enumerate(sweep):
            call(B, k * len(sweep) + j, cfgs[B])

    ev0, ev1 = rt.Event(), rt.Event()
    # Clocks are sampled from the warm-up through the per-batch timings (all
    # under kernel load): the headline region alone is shorter than the
    # sampling period at small --steps.
    clk = ClockSampler(dev).__enter__()
    for k in range(args.warmup):
        step(k)
    ctx.sync()

    # ---- headline timed region ----
    launches0 = ctx.launch_count()
    # DFK_PROFILE_TIMED=1: cudaProfilerStart/Stop around exactly this region,
    # so `ncu --profile-from-start off` lists the timed launches only
    # (tools/profile_round.sh); no effect on the timing otherwise.
    prof = os.environ.get("DFK_PROFILE_TIMED") == "1"
    barrier()
    ctx.sync()
    if prof:
        ctx.profiler_range(True)
    ev0.record(ctx)
    for k in range(args.steps):
        step(k)
    ev1.record(ctx)
    ctx.sync()
    if prof:
        ctx.profiler_range(False)
    barrier()
    ms_total = max_over_ranks(ev0.elapsed_ms(ev1))
    launches = ctx.launch_count() - launches0
    bytes_step = sum(block_bytes(B, DM, DF, P) for B in sweep) * P
    value = bytes_step * args.steps / (ms_total * 1e-3) / 1e9
    ms_per_step = ms_total / args.steps

    # ---- per-batch µs/call (fused, scheduler pick) and the unfused comparator ----
    def time_calls(B, cfg, n, fn=None):
        for i in range(len(sets)):  # touch every weight set (lazy comparator prep)
            (fn or call)(B, i, cfg)
        barrier()
        ctx.sync()
        ev0.record(ctx)
        for i in range(n):
            (fn or call)(B, i, cfg)
        ev1.record(ctx)
        ctx.sync()
        return max_over_ranks(ev0.elapsed_ms(ev1)) * 1e3 / n

    n_rep = max(args.steps, 10)
    us = {B: time_calls(B, cfgs[B], n_rep) for B in sweep}
    two = rt.Config.make(variant=rt.VARIANT_TWO_KERNEL)
    # unfused = cuBLASLt two-kernel layout (+ NCCL's all-reduce under TP; the
    # fused TP path always runs the block kernel)
    nccl_ok = P > 1 and not args.tp_emulate
    us_unfused = ({B: time_calls(B, two, n_rep, nccl_call if P > 1 else None) for B in sweep}
                  if P == 1 or nccl_ok else {B: float("nan") for B in sweep})
    # TP: the same block with NCCL's all-reduce as a separate collective.
    us_nccl = ({B: time_calls(B, cfgs[B], n_rep, nccl_call) for B in sweep}
               if tp_mode == "fused-nvlink" and nccl_ok else None)

    # ---- roofline: the dominant kernel alone ----
    # Block kernel chosen -> the whole block is one launch; otherwise the fused
    # stage-1 kernel (2/3 of the bytes) is the dominant launch.
    a2s = {B: ctx.array((B, f1 - f0)) for B in sweep}
    dom_block = {B: bool(cfgs[B].block_kernel) and cfgs[B].variant == rt.VARIANT_FUSED
                 for B in sweep}

    def dom_call(B, i, cfg):
        if dom_block[B]:
            ctx.forward(sets[i % len(sets)], xs[B], ys[B], cfg=cfg)
        else:
            s1cfg = cfg if cfg.variant == rt.VARIANT_FUSED else rt.Config.make()
            ctx.stage1(sets[i % len(sets)], xs[B], a2s[B], cfg=s1cfg)

    s1_us = {B: time_calls(B, cfgs[B], n_rep, dom_call) for B in sweep}
    clk.__exit__(None, None, None)
    s1_bytes = {B: (block_bytes(B, DM, DF, P) if dom_block[B] else
                    2 * (B * DM + 2 * DM * (f1 - f0) + B * (f1 - f0))) for B in sweep}
    s1_achieved = sum(s1_bytes.values()) / (sum(s1_us.values()) * 1e-6) / 1e9
    dom_name = ("fused block kernel (stream_kernel<kModeBlock>)" if all(dom_block.values())
                else "fused stage-1 kernel (stream_kernel<kModeStage1>)"
                if not any(dom_block.values()) else
                "per batch: block kernel where chosen, else fused stage-1 kernel")
    peak, peak_src = measured_peak()
    floor = stream_floor() if P == 1 else None
    traffic = None
    # DRAM bytes per launch of the dominant kernel from the committed ncu
    # --set full capture (tools/ncu_summary.py traffic), averaged over the sweep.
    tp = os.path.join(ROOT, "profiles", "block_traffic.json")
    if os.path.exists(tp) and all(dom_block.values()) and P == 1:
        try:
            traffic = json.load(open(tp)).get("dram_bytes_per_launch_sweep_mean")
        except Exception:
            traffic = None

    # ---- e2e through the host-buffer C-ABI call ----
    hx = {B: rt.PinnedHost((B, DM), np.uint16) for B in sweep}
    hy = {B: rt.PinnedHost((B, DM), np.float32) for B in sweep}
    for B in sweep:
        hx[B].arr[...] = xs[B].download_bits()

    def host_call(B, i, cfg):
        ctx.forward_host_async(sets[i % len(sets)], hx[B].arr, hy[B].arr, cfg=cfg)

    for k in range(2):
        for B in sweep:
            host_call(B, k, cfgs[B])
    barrier()
    ctx.sync()
    e2e_steps = max(3, args.steps // 2)
    t0 = time.perf_counter()
    ev0.record(ctx)
    for k in range(e2e_steps):
        # one step = every batch of the sweep: H2D of its X from pinned host
        # memory, the block, D2H of its Y; the host waits for the step's
        # results before starting the next step.
        for j, B in enumerate(sweep):
            host_call(B, k * len(sweep) + j, cfgs[B])
        ctx.sync()
    ev1.record(ctx)
    ctx.sync()
    wall = time.perf_counter() - t0
    e2e_ms = max_over_ranks(max(ev0.elapsed_ms(ev1), wall * 1e3))
    e2e = bytes_step * e2e_steps / (e2e_ms * 1e-3) / 1e9

    # ---- isolated single-call latency: L2 flushed, no PDL partner ----
    # (the headline µs/call are back-to-back PDL-chained blocks, whose weight
    # prefetch overlaps the previous block's tail; a decoder with attention
    # between MLP blocks sees this number instead)
    iso = {}
    if P == 1:
        for B in sweep:
            v = []
            for i in range(5):
                ctx.flush_l2()
                ev0.record(ctx)
                ctx.forward(sets[i % len(sets)], xs[B], ys[B], cfg=cfgs[B])
                ev1.record(ctx)
                ctx.sync()
                v.append(ev0.elapsed_ms(ev1) * 1e3)
            iso[str(B)] = round(statistics.median(v), 2)

    # ---- the reference-facing host call with fp64 in/out (dfk_forward_host:
    # fp64 -> bf16 X on the host, H2D, block, D2H, fp32 -> fp64 Y; what the
    # C++ drop-in's run_fused(Matrix) pays per call), synchronous ----
    f64_host = {}
    if P == 1:
        for B in sweep:
            xh = np.random.default_rng(B).uniform(-1, 1, (B, DM))
            ctx.forward_host(sets[0], xh, cfg=cfgs[B])
            v = []
            for i in range(5):
                t0 = time.perf_counter()
                ctx.forward_host(sets[i % len(sets)], xh, cfg=cfgs[B])
                v.append((time.perf_counter() - t0) * 1e6)
            f64_host[str(B)] = round(statistics.median(v), 1)

    # ---- the reference operator API through the C++ drop-in (fp64 Matrix in
    # and out, tools/shim_timing): warm calls, weights cached by Matrix
    # id + version after the first call ----
    shim = None
    exe = os.path.join(ROOT, "tools", "shim_timing")
    if P == 1 and os.path.exists(exe):
        try:
            out = subprocess.run([exe], capture_output=True, text=True, timeout=300).stdout
            shim = [json.loads(ln) for ln in out.splitlines() if ln.startswith("{")] or None
        except Exception:  # noqa: BLE001
            shim = None

    # ---- config 3: multi-layer decode loop (bench.cpp:98-115), CUDA graph ----
    decode = None
    if P == 1 and not args.no_decode:
        decode = decode_loop(rt, ctx, ev0, ev1)
    shards = None
    if P == 1 and not args.no_tp_shards:
        shards = tp_shards(rt, ctx, ev0, ev1, tune=not args.no_tune)
    tp_full = None
    if P > 1 and not args.no_tp_shards and not args.tp_emulate:
        tp_full = tp_configs(rt, ctx, ev0, ev1, rank, P, tp_mode, barrier, max_over_ranks)

    parity = None
    pe = os.path.join(ROOT, "profiles", "r2_parity_errors.json")
    if os.path.exists(pe):
        try:
            parity = json.load(open(pe))
            parity["source"] = "profiles/r2_parity_errors.json (tests/test_gpu_parity.py::test_llama8b_error_report)"
        except Exception:  # noqa: BLE001
            parity = None

    # ---- CPU baseline: reference path, rank 0, N=1 only ----
    cpu = None
    if rank == 0 and P == 1 and not args.no_cpu:
        try:
            gbs, n, per = CpuReference(B=1).time(threads=1, budget_s=12.0)
            cpu = {"value": round(gbs, 4), "unit": "GB/s", "cores": 1, "kind": "reference",
                   "sample": f"reference run_fused as shipped (1 worker, fused.cpp:252), "
                             f"Llama-8B B=1, fp64, median of {n} calls "
                             f"({per * 1e3:.1f} ms/call)",
                   "cpu_model": _cpu_model(), "host_threads": os.cpu_count()}
        except Exception as e:  # noqa: BLE001
            cpu = {"value": None, "unit": "GB/s", "cores": 1, "kind": "reference",
                   "sample": f"unavailable: {e}"}

    if rank == 0:
        line = {
            "metric": METRIC, "value": round(value, 2), "unit": "GB/s", "n_gpus": P,
            "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": round(ms_per_step, 4), "higher_is_better": True,
            "scaling": "strong" if P > 1 else "weak", "vs_baseline": None,
            "dtype": "bf16", "data": "synthetic (uniform bf16, device-generated)",
            "config": {"workload": WORKLOAD, "batch_sweep": sweep, "d_model": DM, "d_ff": DF,
                       "parallelism": f"tp{P}" if P > 1 else "single-gpu",
                       "weight_sets": args.sets,
                       "l2": "inputs larger than L2: 352 MB per weight set, "
                             f"{args.sets} sets rotated", "kernels": "scheduler-selected"},
            "us_per_call": {str(B): round(us[B], 2) for B in sweep},
            "tokens_per_s": {str(B): round(B / (us[B] * 1e-6), 1) for B in sweep},
            "gbs_per_batch": {str(B): round(block_bytes(B, DM, DF, P) * P / (us[B] * 1e-6) / 1e9, 1)
                              for B in sweep},
            "unfused_us_per_call": {str(B): round(us_unfused[B], 2) for B in sweep},
            "tp_allreduce": tp_mode,
            "tp_fused_check": fused_check,
            "nccl_allreduce_us_per_call": ({str(B): round(us_nccl[B], 2) for B in sweep}
                                           if us_nccl else None),
            "speedup_vs_unfused": {str(B): round(us_unfused[B] / us[B], 3) for B in sweep},
            "chosen": chosen,
            "roofline": {"bound": "hbm", "achieved": round(s1_achieved, 1), "peak": peak,
                         "unit": "GB/s", "frac": round(s1_achieved / peak, 4),
                         "traffic": traffic, "kernel": dom_name,
                         "peak_source": peak_src,
                         "stream_floor": floor,
                         "frac_of_stream_floor": (round(s1_achieved / floor["gbs"], 4)
                                                  if floor else None),
                         "per_batch_us": {str(B): round(s1_us[B], 2) for B in sweep}},
            "e2e": {"value": round(e2e, 2), "unit": "GB/s",
                    "h2d_bytes_per_step": sum(B * DM * 2 for B in sweep),
                    "d2h_bytes_per_step": sum(B * DM * 4 for B in sweep)},
            "isolated_us_per_call": iso or None,
            "e2e_f64_host_us_per_call": f64_host or None,
            "reference_api_us_per_call": shim,
            "parity_errors": parity,
            "gpu_launches": int(launches),
            "clocks": clk.summary(),
            "cpu_baseline": cpu,
            "decode_loop": decode,
            "tp_rank_blocks": shards,
            "tp_configs": tp_full,
        }
        print(json.dumps(line), flush=True)
    barrier()
    if dist:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
