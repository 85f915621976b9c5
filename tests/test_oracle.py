"""CPU tests: the oracle (oracle/dfk_oracle.c) pinned against the reference.

The reference library (oracle/_ref/libdeepfusion_ref.so) is the unmodified
/root/reference/proj/src compiled by oracle/Makefile; the golden vectors in
tests/golden/golden.npz were generated from it by tests/golden/make_golden.py.
"""
import hashlib

import numpy as np
import pytest


def _digest(*arrs):
    h = hashlib.sha256()
    for a in arrs:
        h.update(np.ascontiguousarray(a, dtype=np.float64).tobytes())
    return h.hexdigest()


def _case(golden, oracle_lib, name):
    seed, B, dm, df, q = (int(v) for v in golden[f"{name}/meta"])
    scale = float(golden[f"{name}/scale"][0])
    x, wu, wg, wd = oracle_lib.make_instance(seed, B, dm, df, scale)
    if q:
        x, wu, wg, wd = (oracle_lib.quantize_bf16(a)[0] for a in (x, wu, wg, wd))
    return x, wu, wg, wd


# --- generator ------------------------------------------------------------------
@pytest.mark.parametrize("seed,shape", [(0, (1, 4, 8)), (21, (3, 5, 7)),
                                        (20260809, (5, 13, 17)), (7, (8, 64, 64))])
def test_generator_matches_reference(oracle_lib, ref_lib, seed, shape):
    """mt19937_64 + uniform_double + fill order (tensor.cpp:151-163,
    swiglu.cpp:41-51, verification.cpp:28-34) are bit-identical."""
    ours = oracle_lib.make_instance(seed, *shape, 0.5)
    theirs = ref_lib.make_instance(seed, *shape, 0.5)
    for a, b in zip(ours, theirs):
        assert np.array_equal(a, b)


def test_golden_inputs_regenerate_bit_exactly(oracle_lib, golden):
    for name in golden["names"]:
        x, wu, wg, wd = _case(golden, oracle_lib, str(name))
        assert _digest(x, wu, wg, wd) == bytes(golden[f"{name}/digest"]).decode(), name


# --- oracle vs reference -------------------------------------------------------
def test_oracle_matches_golden_vectors(oracle_lib, golden):
    """The C restatement reproduces the reference outputs: bit-exact vs the
    reference oracle_forward, <= 1e-10 vs run_fused (verification.cpp:217-254)."""
    for name in golden["names"]:
        name = str(name)
        x, wu, wg, wd = _case(golden, oracle_lib, name)
        a2, y = oracle_lib.forward(x, wu, wg, wd)
        assert np.abs(a2 - golden[f"{name}/a2"]).max() <= 1e-10, name
        assert np.abs(y - golden[f"{name}/y"]).max() <= 1e-10, name
        if f"{name}/y_oracle" in golden:
            assert np.array_equal(y, golden[f"{name}/y_oracle"]), name


def test_oracle_bit_exact_vs_reference_oracle(oracle_lib, ref_lib):
    rng = np.random.default_rng(5)
    for trial in range(20):
        B, dm, df = (int(v) for v in (rng.integers(1, 9), rng.integers(2, 65),
                                      rng.integers(2, 65)))
        x, wu, wg, wd = ref_lib.make_instance(1000 + trial, B, dm, df)
        a2r, yr = ref_lib.instance(x, wu, wg, wd).oracle_forward()
        a2, y = oracle_lib.forward(x, wu, wg, wd)
        assert np.array_equal(a2, a2r) and np.array_equal(y, yr)


def test_oracle_thread_count_invariance(oracle_lib):
    x, wu, wg, wd = oracle_lib.make_instance(3, 4, 96, 160, 0.1)
    saved = oracle_lib.threads
    try:
        oracle_lib.threads = 1
        a, y1 = oracle_lib.forward(x, wu, wg, wd)
        oracle_lib.threads = 7
        b, y7 = oracle_lib.forward(x, wu, wg, wd)
    finally:
        oracle_lib.threads = saved
    assert np.array_equal(a, b) and np.array_equal(y1, y7)


# --- known answers -------------------------------------------------------------
def test_scalar_known_answer(oracle_lib, golden):
    """x=2, W_up=3, W_gate=1, W_down=1 -> 6*silu(2) = 10.5696
    (test_swiglu.cpp:65-76; SPEC.md's 5.2846 is wrong)."""
    one = np.ones((1, 1))
    _, y = oracle_lib.forward(2 * one, 3 * one, one, one)
    assert abs(y[0, 0] - golden["kat_scalar/y"][0, 0]) <= 1e-15
    assert abs(y[0, 0] - 10.5696) < 1e-4


def test_silu_frozen_values(oracle_lib, golden):
    """test_tensor.cpp:115-128."""
    s1, s0, sm50, s2 = golden["kat_silu"]
    assert oracle_lib.silu(1.0) == s1 == pytest.approx(0.7310585786300049, abs=1e-15)
    assert oracle_lib.sigmoid(0.0) == 0.5 and oracle_lib.silu(0.0) == s0 == 0.0
    assert abs(oracle_lib.silu(-50.0)) <= 1e-15
    assert oracle_lib.silu(2.0) == s2
    for v in np.linspace(-20, 20, 81):
        assert abs(oracle_lib.silu(v) - oracle_lib.silu(-v) - v) <= 1e-12


def test_zero_input_and_zero_gate(oracle_lib):
    """test_swiglu.cpp:46-63."""
    x, wu, wg, wd = oracle_lib.make_instance(3, 1, 3, 4)
    _, y = oracle_lib.forward(np.zeros_like(x), wu, wg, wd)
    assert not y.any()
    x = np.array([[1.0, 0.0]])
    _, y = oracle_lib.forward(x, np.ones((2, 2)), np.zeros((2, 2)), np.eye(2))
    assert not y.any()


def test_bf16_quantisation_is_rne(oracle_lib):
    v = np.array([1.0, 1.0 + 2 ** -8, 1.0 + 3 * 2 ** -8, -2.5, 3.0e-3, 0.0])
    q, bits = oracle_lib.quantize_bf16(v)
    assert q[0] == 1.0 and q[1] == 1.0          # tie -> even
    assert q[2] == 1.0 + 2 ** -6                  # tie -> even (up)
    assert q[3] == -2.5 and q[5] == 0.0
    assert bits[0] == 0x3F80
    assert np.array_equal(oracle_lib.bf16_to_double(bits), q)


# --- TP / traffic --------------------------------------------------------------
def test_balanced_ranges_match_reference(oracle_lib, ref_lib):
    for extent, parts in [(8, 4), (7, 3), (14336, 8), (18944, 8), (5, 5), (100, 7)]:
        assert oracle_lib.balanced_ranges(extent, parts) == \
            ref_lib.balanced_ranges(extent, parts)
    for extent, parts in [(3, 4), (5, 0)]:
        with pytest.raises(ValueError):
            oracle_lib.balanced_ranges(extent, parts)
        with pytest.raises(ValueError):
            ref_lib.balanced_ranges(extent, parts)


def test_tp_sum_in_device_order_matches_golden(oracle_lib, golden):
    """Per-shard oracle partials summed in device order reproduce the
    reference's run_tp_mlp (tp.cpp:140-167) for P in {1,2,3,4,8}."""
    for name in ("tp_3x6x12", "uneven_2x4x7"):
        x, wu, wg, wd = _case(golden, oracle_lib, name)
        df = wu.shape[1]
        for P in (1, 2, 3, 4, 8):
            key = f"{name}/tp{P}"
            if key not in golden:
                continue
            parts = []
            for b, e in oracle_lib.balanced_ranges(df, P):
                _, yp = oracle_lib.forward(x, np.ascontiguousarray(wu[:, b:e]),
                                           np.ascontiguousarray(wg[:, b:e]),
                                           np.ascontiguousarray(wd[b:e, :]))
                parts.append(yp)
            y = oracle_lib.allreduce_in_order(np.stack(parts))
            assert np.abs(y - golden[key]).max() <= 1e-12
            ev, payload = golden[f"{key}_log"]
            assert ev == 1 and payload == x.shape[0] * x.shape[1]


def test_fused_block_bytes_match_traffic_model(oracle_lib, ref_lib):
    """Algorithmic bytes = predict_traffic(Fused, single tile) at 2 B/elem
    (traffic.cpp:70-76, 82-94)."""
    for B, dm, df in [(1, 4096, 14336), (16, 4096, 14336), (64, 8192, 3584),
                      (2, 4, 8), (7, 3584, 18944)]:
        assert oracle_lib.fused_block_bytes(B, dm, df) == ref_lib.fused_block_bytes(B, dm, df)
    # Llama-3.1-8B B=1 per-call bytes.
    assert oracle_lib.fused_block_bytes(1, 4096, 14336) == 352_395_264
