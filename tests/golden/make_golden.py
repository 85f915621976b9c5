"""Generate the golden vectors in tests/golden/golden.npz from the REFERENCE.

Run in the build container (needs oracle/_ref/libdeepfusion_ref.so, i.e. the
unmodified reference compiled from /root/reference/proj/src by oracle/Makefile):

    python tests/golden/make_golden.py

Every case stores its generator parameters (seed, shape, scale), whether the
inputs were rounded to bf16 (the GPU's input type), a SHA-256 of the input
bits, and the reference outputs: A2 from ``run_fused_stage1`` and Y from
``run_fused`` (``fused.cpp:172-216``) with a single covering column-major
tile, plus ``oracle_forward`` (``verification.cpp:188-202``).  Inputs are
regenerated at test time from the seed, so the fixture stays small.

Generator: the reference's ``make_random_weights`` + ``fill_uniform``
(``swiglu.cpp:41-51``, ``tensor.cpp:151-163``): W_up, W_gate, W_down, then X.
"""
import hashlib
import os
import sys

import numpy as np

sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", ".."))
import oracle  # noqa: E402

# (name, seed, B, d_model, d_ff, scale, bf16-quantised inputs)
CASES = [
    ("tiny_3x5x7", 21, 3, 5, 7, 1.0, False),       # test_fused.cpp:47-56 shape/seed
    ("edge_5x7x11", 29, 5, 7, 11, 1.0, False),     # test_fused.cpp:83-93 shape
    ("crit2_5x13x17", 20260809, 5, 13, 17, 1.0, False),  # verification.cpp:278-308 shape
    ("tp_3x6x12", 71, 3, 6, 12, 1.0, False),       # test_tp.cpp:74-89 shape/seed
    ("uneven_2x4x7", 73, 2, 4, 7, 1.0, False),     # test_tp.cpp:91-112 shape/seed
    ("bf16_1x64x128", 1, 1, 64, 128, 0.125, True),
    ("bf16_4x256x512", 2, 4, 256, 512, 1 / 16, True),
    ("bf16_8x512x1536", 3, 8, 512, 1536, 1 / 22.6, True),
    ("bf16_16x128x448", 4, 16, 128, 448, 1 / 11.3, True),
    ("bf16_3x200x300", 5, 3, 200, 300, 1 / 14.1, True),
    ("bf16_64x512x768", 6, 64, 512, 768, 1 / 22.6, True),
]


def input_digest(*arrs):
    h = hashlib.sha256()
    for a in arrs:
        h.update(np.ascontiguousarray(a, dtype=np.float64).tobytes())
    return h.hexdigest()


def main():
    o = oracle.Oracle()
    ref = oracle.Reference()
    out = {}
    names = []
    for name, seed, B, dm, df, scale, q in CASES:
        x, wu, wg, wd = ref.make_instance(seed, B, dm, df, scale)
        if q:
            x, _ = o.quantize_bf16(x); wu, _ = o.quantize_bf16(wu)
            wg, _ = o.quantize_bf16(wg); wd, _ = o.quantize_bf16(wd)
        inst = ref.instance(x, wu, wg, wd)
        a2 = inst.run_fused_stage1()
        y = inst.run_fused()
        a2o, yo = inst.oracle_forward()
        meta = np.array([seed, B, dm, df, int(q)], dtype=np.int64)
        out[f"{name}/meta"] = meta
        out[f"{name}/scale"] = np.array([scale])
        out[f"{name}/digest"] = np.frombuffer(
            input_digest(x, wu, wg, wd).encode(), dtype=np.uint8)
        out[f"{name}/a2"] = a2
        out[f"{name}/y"] = y
        if not q:
            out[f"{name}/y_oracle"] = yo
        names.append(name)
        if name.startswith("tp_") or name.startswith("uneven_"):
            for P in (1, 2, 3, 4, 8) if df >= 8 else (1, 2, 3):
                yt, ev, pl = inst.run_tp_mlp(P, "fused")
                out[f"{name}/tp{P}"] = yt
                out[f"{name}/tp{P}_log"] = np.array([ev, pl], dtype=np.int64)
    # Scalar known answer (test_swiglu.cpp:65-76, test_fused.cpp:179-189):
    # x=2, W_up=3, W_gate=1, W_down=1 -> 6*silu(2) = 10.5696.
    one = np.ones((1, 1))
    inst = ref.instance(2 * one, 3 * one, one, one)
    out["kat_scalar/y"] = inst.run_fused()
    out["kat_silu"] = np.array([ref.silu(1.0), ref.silu(0.0), ref.silu(-50.0),
                                ref.silu(2.0)])
    out["names"] = np.array(names)
    path = os.path.join(os.path.dirname(__file__), "golden.npz")
    np.savez_compressed(path, **out)
    print(f"wrote {path} ({os.path.getsize(path)} bytes, {len(names)} cases)")


if __name__ == "__main__":
    main()
