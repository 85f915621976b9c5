"""Host-side conversions of the reference-facing calls (dfk_host_to_bf16 /
dfk_host_from_f32 / dfk_host_from_bf16, csrc/host_convert.cpp): the fp64
Matrix operands of the reference API (tensor.hpp:73-128) rounded to bf16
bits exactly as the oracle quantises them (fp64 -> fp32 -> bf16 RNE,
oracle/dfk_oracle.c), and widened back exactly.  CPU only (no GPU calls)."""
import threading

import numpy as np
import pytest


@pytest.fixture(scope="module")
def rt():
    from paper_2602_11808_b200 import runtime
    return runtime


def _to_bf16(rt, a, dtype):
    out = np.empty(a.size, dtype=np.uint16)
    rt._check(rt.lib.dfk_host_to_bf16(a.ctypes.data, dtype, a.size, out.ctypes.data))
    return out


def _special_values():
    f = np.array([0.0, -0.0, 1.0, -1.0, np.inf, -np.inf, 1e-40, -1e-40, 3.0e38, 1.5,
                  np.float32(1.00390625), np.float32(1.01171875), 65504.0, 2.0 ** -126],
                 dtype=np.float64)
    # exact ties between two bf16 values: round to even
    ties = np.array([1.0 + 2.0 ** -8, 1.0 + 3 * 2.0 ** -8, -(1.0 + 2.0 ** -8)], dtype=np.float64)
    return np.concatenate([f, ties])


@pytest.mark.parametrize("n", [7, 1000, 300_001, 1_300_007])  # the last: worker pool
def test_f64_to_bf16_matches_oracle(rt, oracle_lib, n):
    rng = np.random.default_rng(n)
    a = rng.standard_normal(n) * np.exp(rng.uniform(-30, 30, n))
    a[: min(n, 17)] = _special_values()[: min(n, 17)]
    got = _to_bf16(rt, a, rt.F64)
    _, want = oracle_lib.quantize_bf16(a)
    assert np.array_equal(got, want)


def test_nan_stays_quiet_nan(rt):
    a = np.array([np.nan, -np.nan, np.float64(np.float32(np.nan))], dtype=np.float64)
    got = _to_bf16(rt, a, rt.F64)
    assert np.all((got & 0x7F80) == 0x7F80) and np.all((got & 0x007F) != 0)
    assert np.all(got & 0x0040)


@pytest.mark.parametrize("n", [5, 200_003, 700_001])
def test_f32_to_bf16_and_bf16_passthrough(rt, oracle_lib, n):
    rng = np.random.default_rng(1 + n)
    f = (rng.standard_normal(n) * 100).astype(np.float32)
    got = _to_bf16(rt, f, rt.F32)
    _, want = oracle_lib.quantize_bf16(f.astype(np.float64))
    assert np.array_equal(got, want)
    assert np.array_equal(_to_bf16(rt, got, rt.BF16), got)


@pytest.mark.parametrize("n", [3, 250_000, 917_504])
def test_widening_is_exact(rt, oracle_lib, n):
    rng = np.random.default_rng(2 + n)
    f = (rng.standard_normal(n) * 1e3).astype(np.float32)
    d = np.empty(n, dtype=np.float64)
    rt._check(rt.lib.dfk_host_from_f32(f.ctypes.data, n, d.ctypes.data, rt.F64))
    assert np.array_equal(d, f.astype(np.float64))
    b = np.empty(n, dtype=np.uint16)
    rt._check(rt.lib.dfk_host_from_f32(f.ctypes.data, n, b.ctypes.data, rt.BF16))
    assert np.array_equal(b, oracle_lib.quantize_bf16(f.astype(np.float64))[1])
    d2 = np.empty(n, dtype=np.float64)
    rt._check(rt.lib.dfk_host_from_bf16(b.ctypes.data, n, d2.ctypes.data, rt.F64))
    assert np.array_equal(d2, oracle_lib.bf16_to_double(b))
    f2 = np.empty(n, dtype=np.float32)
    rt._check(rt.lib.dfk_host_from_bf16(b.ctypes.data, n, f2.ctypes.data, rt.F32))
    assert np.array_equal(f2.astype(np.float64), d2)


def test_concurrent_callers_share_the_pool(rt, oracle_lib):
    """Several host threads converting at once: small calls inline, large
    ones on the worker pool (one job at a time; a caller finding it busy
    converts inline) -- every result exact."""
    rng = np.random.default_rng(9)
    arrays = [rng.standard_normal((180_000 if i % 2 else 700_000) + 1000 * i) for i in range(6)]
    wants = [oracle_lib.quantize_bf16(a)[1] for a in arrays]
    results = [None] * len(arrays)

    def work(i):
        for _ in range(5):
            results[i] = _to_bf16(rt, arrays[i], rt.F64)

    ts = [threading.Thread(target=work, args=(i,)) for i in range(len(arrays))]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    for got, want in zip(results, wants):
        assert np.array_equal(got, want)


def test_bad_arguments(rt):
    a = np.zeros(4)
    assert rt.lib.dfk_host_to_bf16(a.ctypes.data, 7, 4, a.ctypes.data) == rt.ERR_INVALID
    assert rt.lib.dfk_host_from_f32(None, 4, a.ctypes.data, rt.F64) == rt.ERR_INVALID
    assert rt.lib.dfk_host_from_bf16(None, 0, None, rt.F64) == rt.OK

