"""CPU tests of the C-ABI library (no GPU needed): it loads, exports every
symbol include/dfk.h declares, and its host-side logic (balanced ranges,
traffic model, config validation, error classes) follows the reference."""
import ctypes as C
import os
import re
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared_symbols():
    text = open(os.path.join(ROOT, "include", "dfk.h")).read()
    return sorted(set(re.findall(r"DFK_API\s+[\w\s\*]+?\b(dfk_\w+)\s*\(", text)))


def test_library_loads_and_exports_every_declared_symbol():
    import paper_2602_11808_b200 as p
    declared = _declared_symbols()
    assert len(declared) >= 40
    nm = subprocess.run(["nm", "-D", "--defined-only", p.library_path()],
                        capture_output=True, text=True, check=True).stdout
    exported = set(re.findall(r"\bT (dfk_\w+)", nm))
    missing = [s for s in declared if s not in exported]
    assert not missing, missing
    # and the Python layer binds exactly those
    from paper_2602_11808_b200 import runtime
    assert sorted(runtime.EXPORTED_SYMBOLS) == declared


def test_library_is_sm100a_only():
    import paper_2602_11808_b200 as p
    out = subprocess.run(["cuobjdump", "--list-elf", p.library_path()],
                         capture_output=True, text=True, check=True).stdout
    archs = set(re.findall(r"sm_\d+a?", out))
    assert archs == {"sm_100a"}, archs


def test_sass_uses_tcgen05_and_tma():
    import paper_2602_11808_b200 as p
    sass = subprocess.run(["cuobjdump", "-sass", p.library_path()],
                          capture_output=True, text=True, check=True).stdout
    for mnemonic in ("UTCHMMA", "UTMALDG", "UBLKCP", "LDTM"):
        assert mnemonic in sass, mnemonic
    assert "HMMA" not in re.sub(r"UTCHMMA", "", sass)  # no legacy mma.sync path


def test_balanced_range_matches_oracle(oracle_lib):
    from paper_2602_11808_b200 import runtime as rt
    for extent, parts in [(8, 4), (7, 3), (14336, 8), (18944, 8), (27648, 8), (100, 7)]:
        ours = [rt.balanced_range(extent, parts, i) for i in range(parts)]
        assert ours == oracle_lib.balanced_ranges(extent, parts)
    with pytest.raises(rt.ShapeError):
        rt.balanced_range(3, 4, 0)
    with pytest.raises(rt.ShapeError):
        rt.balanced_range(3, 0, 0)


def test_block_bytes_match_traffic_model(oracle_lib):
    from paper_2602_11808_b200 import block_bytes
    for B, dm, df in [(1, 4096, 14336), (16, 4096, 14336), (64, 5120, 3456), (3, 5, 7)]:
        s1, s2 = block_bytes(B, dm, df)
        assert s1 + s2 == oracle_lib.fused_block_bytes(B, dm, df)
    from paper_2602_11808_b200 import ShapeError
    with pytest.raises(ShapeError):
        block_bytes(0, 4, 4)


def test_no_gpu_calls_fail_loudly_not_silently():
    """Without a GPU every compute entry point must return an error (there is
    no CPU fallback)."""
    from paper_2602_11808_b200 import runtime as rt
    if rt.lib.dfk_device_count(C.byref(C.c_int())) == 0:
        n = C.c_int()
        rt.lib.dfk_device_count(C.byref(n))
        if n.value > 0:
            pytest.skip("GPU present")
    with pytest.raises((rt.DfkError, rt.InvalidArgument)):
        rt.Context(0)


def test_bf16_host_rounding_matches_oracle(oracle_lib):
    from paper_2602_11808_b200.runtime import bf16_bits_to_f32, to_bf16_bits
    v = np.random.default_rng(0).standard_normal(4096) * 3
    q, bits = oracle_lib.quantize_bf16(v)
    assert np.array_equal(to_bf16_bits(v), bits)
    assert np.array_equal(bf16_bits_to_f32(bits).astype(np.float64), q)


def test_mirror_api_validation_without_gpu():
    from paper_2602_11808_b200 import deepfusion as df
    with pytest.raises(df.ShapeError):
        df.TileConfig(0, 1, 1).validate()
    with pytest.raises(df.ShapeError):
        df.MlpShape(0, 4, 4).validate()
    w = df.MlpWeights(np.zeros((4, 8)), np.zeros((4, 8)), np.zeros((8, 3)),
                      df.MlpShape(1, 4, 8))
    with pytest.raises(df.ShapeError):
        w.validate()
    plan = df.ShardPlan(2, [df.ColRange(0, 3), df.ColRange(4, 8)])
    with pytest.raises(df.ShapeError):
        plan.validate(8)
    assert df.TileConfig(2, 3, 4, df.LoopOrder.RowMajorTiling).describe() == "m2_n3_k4_row"
    log = df.CollectiveLog([df.CollectiveEvent(df.CollectiveKind.AllReduce, 4096)])
    assert df.comm_volume_bytes(log, 4, df.CommModel.Logical) == 8192
    assert df.comm_volume_bytes(log, 4, df.CommModel.Ring) == pytest.approx(2 * 3 / 4 * 8192)


def test_tune_front_end_usage_errors_exit_2():
    """The `tune` front end keeps the reference CLI's exit contract
    (main.cpp:377-389): usage errors -> 2 (checked without a GPU: argument
    validation happens before any device work)."""
    from paper_2602_11808_b200 import tune
    assert tune.main(["--batch", "1,x"]) == 2
    assert tune.main(["--no-such-flag"]) == 2
    assert tune.resolve_cache_path("a.json") == "a.json"
    os.environ["DEEPFUSION_CACHE"] = "env.json"
    try:
        assert tune.resolve_cache_path("") == "env.json"
    finally:
        del os.environ["DEEPFUSION_CACHE"]
    assert tune.resolve_cache_path("") == "deepfusion_cache.json"
