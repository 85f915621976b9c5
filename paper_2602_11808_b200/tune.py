"""`tune` front end: the reference CLI's `deepfusion tune` (tools/main.cpp
run_tune :210-236) over the GPU scheduler (dfk_tune).

    python -m paper_2602_11808_b200.tune --d-model 4096 --d-ff 14336 \\
        --batch 1,2,4,8,16 [--cache-path P] [--warmup 1] [--runs 4] [--seed 0] [--tp 1]

Per batch size: get-or-tune the (B, d_model, d_ff shard) key against the JSON
cache (format_version 1, flock-guarded), print
``B=.. d_model=.. d_ff=.. -> <label> (cache hit, profiling skipped|profiled)``
and the count of candidates the correctness gate disqualified; finally
``cache: <path> [<fingerprint>]``.  Cache path: --cache-path, else
$DEEPFUSION_CACHE, else ./deepfusion_cache.json (main.cpp:62-66).  Exit codes
as the reference CLI (main.cpp:377-389): 0 ok, 2 usage / shape errors, 1
anything else.  --tp P tunes rank 0's balanced_ranges shard of d_ff (the
fingerprint carries the TP degree).  Weights are synthetic bf16
U[-1/sqrt(d_model), 1/sqrt(d_model)), generated on the device.
"""
from __future__ import annotations

import argparse
import os
import sys

EXIT_OK, EXIT_FAIL, EXIT_USAGE = 0, 1, 2
CACHE_ENV = "DEEPFUSION_CACHE"


def resolve_cache_path(flag: str) -> str:
    if flag:
        return flag
    return os.environ.get(CACHE_ENV) or "deepfusion_cache.json"


def parse_index_list(text: str, flag: str):
    try:
        out = [int(v) for v in text.split(",") if v.strip()]
    except ValueError:
        raise ValueError(f"{flag}: expected a comma-separated int list") from None
    if not out:
        raise ValueError(f"{flag}: expected a non-empty list")
    return out


def run_tune(args) -> int:
    from . import runtime as rt

    batches = parse_index_list(args.batch, "--batch")
    if args.d_model < 1 or args.d_ff < 1 or any(b < 1 for b in batches) or args.tp < 1:
        raise rt.ShapeError("dims, batch sizes and --tp must be >= 1")
    ratio = args.d_ff / args.d_model
    if not 3.5 <= ratio <= 4.0:
        print(f"note: d_ff/d_model = {ratio:g} is outside the usual [3.5, 4.0] band",
              file=sys.stderr)
    cache = resolve_cache_path(args.cache_path)
    ctx = rt.Context(0)
    b0, b1 = rt.balanced_range(args.d_ff, args.tp, 0)
    s = 1.0 / args.d_model ** 0.5
    g = ctx.array((args.d_model, args.d_ff)).fill_uniform(args.seed * 3 + 1, -s, s)
    u = ctx.array((args.d_model, args.d_ff)).fill_uniform(args.seed * 3 + 2, -s, s)
    d = ctx.array((args.d_ff, args.d_model)).fill_uniform(args.seed * 3 + 3, -s, s)
    w = ctx.weights(g, u, d, ff_range=(b0, b1))
    del g, u, d
    for B in batches:
        cfg, hit, entry = ctx.tune(w, B, cache, args.warmup, args.runs)
        print(f"B={B} d_model={args.d_model} d_ff={args.d_ff} -> {cfg.label.decode()}"
              f" ({'cache hit, profiling skipped' if hit else 'profiled'})")
        dq = sum(1 for r in entry.get("results", []) if r.get("disqualified"))
        if dq:
            print(f"  {dq} candidate(s) disqualified by the correctness gate")
    print(f"cache: {cache} [{ctx.fingerprint()}]")
    return EXIT_OK


def main(argv=None) -> int:
    ap = argparse.ArgumentParser(prog="tune", description=__doc__.split("\n")[0])
    ap.add_argument("--d-model", type=int, default=512)
    ap.add_argument("--d-ff", type=int, default=2048)
    ap.add_argument("--batch", default="1,2,4,8")
    ap.add_argument("--warmup", type=int, default=1)
    ap.add_argument("--runs", type=int, default=4)
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--tp", type=int, default=1)
    ap.add_argument("--cache-path", default="")
    try:
        args = ap.parse_args(argv)
    except SystemExit as e:  # argparse: usage errors exit 2 already
        return int(e.code or 0)
    from . import runtime as rt
    try:
        return run_tune(args)
    except (ValueError, rt.ShapeError, rt.InvalidArgument) as e:
        print(f"error: {e}", file=sys.stderr)
        return EXIT_USAGE
    except Exception as e:  # noqa: BLE001  (main.cpp: anything else -> 1)
        print(f"error: {e}", file=sys.stderr)
        return EXIT_FAIL


if __name__ == "__main__":
    sys.exit(main())
