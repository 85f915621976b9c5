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
