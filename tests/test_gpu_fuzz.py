"""Randomised parity sweep of the default configuration (the scheduler's
NULL config -> block kernel with the dynamic queue) over ragged shapes:
d_model / d_ff not multiples of the 64 / 128 tiles, d_ff on both sides of
the full-stage-1-wave threshold (64 x SMs), B across every MMA width and the
256-row chunking.  Each instance: the forward twice back to back, then the
separate stage-1 + down entry points, all against the fp64 oracle."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

TOL = 1e-2


def rel_err(got, ref):
    den = np.abs(ref).max()
    return float(np.abs(np.asarray(got, np.float64) - ref).max() / (den if den > 0 else 1.0))


def test_random_shapes_default_config(oracle_lib):
    from paper_2602_11808_b200 import runtime as rt

    rng = np.random.default_rng(20261017)
    ctx = rt.Context(0)
    try:
        for case in range(24):
            dm = int(rng.choice([72, 136, 520, 1000, 1544]))
            df = int(rng.choice([100, 1032, 4000, 9500, 9990]))
            B = int(rng.choice([1, 3, 8, 15, 17, 31, 40, 64, 65, 130, 257]))
            x, wu, wg, wd = (oracle_lib.quantize_bf16(a)[0] for a in
                             oracle_lib.make_instance(1000 + case, B, dm, df, 1.0 / np.sqrt(dm)))
            a2_ref, y_ref = oracle_lib.forward(x, wu, wg, wd)
            w = ctx.weights(wg, wu, wd)
            xd = ctx.array((B, dm)).upload(x)
            y = ctx.array((B, dm), rt.F32)
            ctx.forward(w, xd, y)
            ctx.forward(w, xd, y)
            assert rel_err(y.download(), y_ref) <= TOL, ("forward", dm, df, B)
            a2 = ctx.array((B, df))
            y2 = ctx.array((B, dm), rt.F32)
            ctx.stage1(w, xd, a2)
            ctx.down(w, a2, y2)
            assert rel_err(a2.download(), a2_ref) <= TOL, ("stage1", dm, df, B)
            assert rel_err(y2.download(), y_ref) <= TOL, ("down", dm, df, B)
            del w
    finally:
        ctx.close()


def test_random_configs_ragged_shapes(oracle_lib):
    """Random points of the scheduler's search space (tail split 0-4 parts,
    CTA count, stage-1 / down chunk, stage size, kernel family at B <= 8, fp32
    or bf16 Y) on ragged shapes, each run twice back to back against the fp64
    oracle: every configuration dfk_tune may pick must be exact to tolerance,
    not only the ones the default takes."""
    from paper_2602_11808_b200 import runtime as rt

    import os
    rng = np.random.default_rng(int(os.environ.get("DFK_FUZZ_SEED", "20261018")))
    ctx = rt.Context(0)
    try:
        for case in range(int(os.environ.get("DFK_FUZZ_CASES", "30"))):
            dm = int(rng.choice([136, 520, 1000]))
            df = int(rng.choice([1032, 4000, 9990]))
            B = int(rng.choice([1, 5, 8, 16, 33, 64]))
            fam = (rt.FAMILY_GEMV if B <= 8 and rng.random() < 0.3 else rt.FAMILY_TC)
            kw = dict(block_kernel=1, dynamic_sched=1, s1_family=fam, down_family=fam,
                      s1_tail=int(rng.integers(0, 5)),
                      s1_ctas=int(rng.choice([0, 3, 17, 100, 148])),
                      chunk_kb=int(rng.choice([0, 3, 8, 24])),
                      s1_chunk_kb=int(rng.choice([0, 0, 5, 16])),
                      kbs=int(rng.choice([0, 2, 3])) if fam == rt.FAMILY_TC else 0)
            cfg = rt.Config.make(**kw)
            y_dt = rt.BF16 if rng.random() < 0.3 else rt.F32
            x, wu, wg, wd = (oracle_lib.quantize_bf16(a)[0] for a in
                             oracle_lib.make_instance(2000 + case, B, dm, df, 1.0 / np.sqrt(dm)))
            _, y_ref = oracle_lib.forward(x, wu, wg, wd)
            w = ctx.weights(wg, wu, wd)
            xd = ctx.array((B, dm)).upload(x)
            y = ctx.array((B, dm), y_dt)
            for _ in range(2):
                ctx.forward(w, xd, y, cfg=cfg)
            tol = TOL if y_dt == rt.F32 else 2 * TOL
            assert rel_err(y.download(), y_ref) <= tol, (case, dm, df, B, kw, y_dt)
            del w
    finally:
        ctx.close()
