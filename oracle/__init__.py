"""CPU oracle for the fused SwiGLU-MLP path — TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py`` (its
``cpu_baseline`` leg and ``--impl reference``) may import this package, and
only as the checker / the timed reference arm.  The product package
``paper_2602_11808_b200`` never imports it and fails loudly when its CUDA
library is missing.

Two layers, both numpy-facing through ctypes:

* :class:`Oracle` wraps ``oracle/liboracle.so`` built from
  ``oracle/dfk_oracle.c`` — a plain-C restatement of the reference's fp64
  oracle (``/root/reference/proj/src/verification.cpp:171-202``), its
  generator (``src/tensor.cpp:151-163``) and ``balanced_ranges``
  (``src/tp.cpp:8-29``).
* :class:`Reference` wraps ``oracle/_ref/libdeepfusion_ref.so`` — the
  unmodified reference library compiled in place by ``oracle/Makefile``
  (plus the ``oracle/ref_capi.cpp`` extern-"C" shim).  It pins the
  restatement (``tests/test_oracle.py``) and is the CPU baseline.

Parity status: pinned (against ``oracle/_ref`` and ``tests/golden/``).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libdeepfusion_ref.so")
REF_SRC = "/root/reference/proj/src"

_f64p = np.ctypeslib.ndpointer(dtype=np.float64, flags="C_CONTIGUOUS")
_u16p = np.ctypeslib.ndpointer(dtype=np.uint16, flags="C_CONTIGUOUS")
_i64p = np.ctypeslib.ndpointer(dtype=np.int64, flags="C_CONTIGUOUS")


def build(quiet: bool = True) -> None:
    """Build liboracle.so and, when /root/reference exists, the _ref library."""
    out = subprocess.DEVNULL if quiet else None
    subprocess.run(["make", "-C", HERE, "-j8", "all"], check=True, stdout=out)


def _load(path: str) -> C.CDLL:
    if not os.path.exists(path):
        if path == ORACLE_SO or os.path.isdir(REF_SRC):
            build()
    if not os.path.exists(path):
        raise FileNotFoundError(f"{path} not built (run `make -C oracle`)")
    return C.CDLL(path)


class Oracle:
    """The C restatement (oracle/dfk_oracle.c)."""

    def __init__(self) -> None:
        lib = _load(ORACLE_SO)
        lib.dfo_make_instance.argtypes = [C.c_uint64, C.c_int64, C.c_int64, C.c_int64,
                                          C.c_double, _f64p, _f64p, _f64p, _f64p]
        lib.dfo_quantize_bf16.argtypes = [_f64p, C.c_void_p, C.c_int64]
        lib.dfo_bf16_to_double.argtypes = [_u16p, _f64p, C.c_int64]
        lib.dfo_silu.argtypes = [C.c_double]
        lib.dfo_silu.restype = C.c_double
        lib.dfo_sigmoid.argtypes = [C.c_double]
        lib.dfo_sigmoid.restype = C.c_double
        lib.dfo_stage1.argtypes = [_f64p, _f64p, _f64p, C.c_int64, C.c_int64, C.c_int64,
                                   _f64p, C.c_int]
        lib.dfo_down.argtypes = [_f64p, _f64p, C.c_int64, C.c_int64, C.c_int64, _f64p,
                                 C.c_int, C.c_int]
        lib.dfo_forward.argtypes = [_f64p, _f64p, _f64p, _f64p, C.c_int64, C.c_int64,
                                    C.c_int64, _f64p, _f64p, C.c_int, C.c_int]
        lib.dfo_allreduce_in_order.argtypes = [_f64p, C.c_int64, C.c_int64, _f64p]
        lib.dfo_balanced_ranges.argtypes = [C.c_int64, C.c_int64, _i64p, _i64p]
        lib.dfo_balanced_ranges.restype = C.c_int
        lib.dfo_fused_block_bytes.argtypes = [C.c_int64, C.c_int64, C.c_int64, C.c_uint64]
        lib.dfo_fused_block_bytes.restype = C.c_uint64
        self.lib = lib
        self.threads = max(1, os.cpu_count() or 1)

    # -- generator --------------------------------------------------------
    def make_instance(self, seed: int, B: int, dm: int, df: int, scale: float = 1.0):
        """(x, w_up, w_gate, w_down) in fp64, reference fill order."""
        x = np.empty((B, dm)); wu = np.empty((dm, df)); wg = np.empty((dm, df))
        wd = np.empty((df, dm))
        self.lib.dfo_make_instance(seed, B, dm, df, scale, x, wu, wg, wd)
        return x, wu, wg, wd

    def quantize_bf16(self, v: np.ndarray):
        """Round to bf16 (via fp32, RNE). Returns (widened fp64, bf16 bits as uint16)."""
        v = np.ascontiguousarray(v, dtype=np.float64).copy()
        bits = np.empty(v.shape, dtype=np.uint16)
        self.lib.dfo_quantize_bf16(v, bits.ctypes.data, v.size)
        return v, bits

    def bf16_to_double(self, bits: np.ndarray) -> np.ndarray:
        bits = np.ascontiguousarray(bits, dtype=np.uint16)
        out = np.empty(bits.shape, dtype=np.float64)
        self.lib.dfo_bf16_to_double(bits, out, bits.size)
        return out

    def silu(self, x: float) -> float:
        return self.lib.dfo_silu(x)

    def sigmoid(self, x: float) -> float:
        return self.lib.dfo_sigmoid(x)

    # -- oracle kernels ---------------------------------------------------
    def stage1(self, x, w_up, w_gate) -> np.ndarray:
        B, dm = x.shape
        df = w_up.shape[1]
        a2 = np.empty((B, df))
        self.lib.dfo_stage1(np.ascontiguousarray(x), np.ascontiguousarray(w_up),
                            np.ascontiguousarray(w_gate), B, dm, df, a2, self.threads)
        return a2

    def down(self, a2, w_down, quant_a2: bool = False) -> np.ndarray:
        B, df = a2.shape
        dm = w_down.shape[1]
        y = np.empty((B, dm))
        self.lib.dfo_down(np.ascontiguousarray(a2), np.ascontiguousarray(w_down), B, df,
                          dm, y, int(quant_a2), self.threads)
        return y

    def forward(self, x, w_up, w_gate, w_down, quant_a2: bool = False):
        """Returns (a2, y) of oracle_forward (verification.cpp:188-202)."""
        B, dm = x.shape
        df = w_up.shape[1]
        a2 = np.empty((B, df)); y = np.empty((B, dm))
        self.lib.dfo_forward(np.ascontiguousarray(x), np.ascontiguousarray(w_up),
                             np.ascontiguousarray(w_gate), np.ascontiguousarray(w_down),
                             B, dm, df, a2, y, int(quant_a2), self.threads)
        return a2, y

    def allreduce_in_order(self, partials: np.ndarray) -> np.ndarray:
        partials = np.ascontiguousarray(partials, dtype=np.float64)
        P = partials.shape[0]
        out = np.empty(partials.shape[1:])
        self.lib.dfo_allreduce_in_order(partials, P, out.size, out)
        return out

    def balanced_ranges(self, extent: int, parts: int):
        b = np.zeros(max(parts, 1), dtype=np.int64); e = np.zeros_like(b)
        if self.lib.dfo_balanced_ranges(extent, parts, b, e) != 0:
            raise ValueError(f"balanced_ranges: cannot split {extent} into {parts}")
        return list(zip(b.tolist(), e.tolist()))

    def fused_block_bytes(self, B: int, dm: int, df: int, bpe: int = 2) -> int:
        return int(self.lib.dfo_fused_block_bytes(B, dm, df, bpe))


class ReferenceError_(RuntimeError):
    pass


class Reference:
    """The unmodified reference library (oracle/_ref/libdeepfusion_ref.so)."""

    VARIANTS = {"four_kernel": 0, "two_kernel": 1, "fused": 2}

    def __init__(self) -> None:
        lib = _load(REF_SO)
        lib.dfr_last_error.restype = C.c_char_p
        lib.dfr_silu.argtypes = [C.c_double]
        lib.dfr_silu.restype = C.c_double
        lib.dfr_make_instance.argtypes = [C.c_uint64, C.c_int64, C.c_int64, C.c_int64,
                                          C.c_double, _f64p, _f64p, _f64p, _f64p]
        lib.dfr_instance_create.argtypes = [C.c_int64, C.c_int64, C.c_int64, _f64p, _f64p,
                                            _f64p, _f64p]
        lib.dfr_instance_create.restype = C.c_void_p
        lib.dfr_instance_destroy.argtypes = [C.c_void_p]
        lib.dfr_run_fused.argtypes = [C.c_void_p, C.c_int64, C.c_int64, C.c_int64, C.c_int,
                                      C.c_int, _f64p]
        lib.dfr_run_fused_stage1.argtypes = lib.dfr_run_fused.argtypes
        lib.dfr_run_variant.argtypes = [C.c_void_p, C.c_int, C.c_int64, C.c_int64,
                                        C.c_int64, C.c_int, _f64p]
        lib.dfr_down_projection.argtypes = [_f64p, C.c_int64, C.c_int64, _f64p, C.c_int64,
                                            _f64p]
        lib.dfr_oracle_forward.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p]
        lib.dfr_run_tp_mlp.argtypes = [C.c_void_p, C.c_int64, C.c_int, _f64p,
                                       C.POINTER(C.c_int64), C.POINTER(C.c_int64)]
        lib.dfr_balanced_ranges.argtypes = [C.c_int64, C.c_int64, _i64p, _i64p]
        lib.dfr_fused_block_bytes.argtypes = [C.c_int64, C.c_int64, C.c_int64, C.c_uint64]
        lib.dfr_fused_block_bytes.restype = C.c_uint64
        lib.dfr_default_candidate_count.argtypes = [C.c_int64, C.c_int64, C.c_int64]
        lib.dfr_default_candidate_count.restype = C.c_int64
        self.lib = lib

    def _check(self, rc: int) -> None:
        if rc != 0:
            msg = self.lib.dfr_last_error().decode()
            if rc == 2:
                raise ValueError(msg)
            raise ReferenceError_(msg)

    def silu(self, x: float) -> float:
        return self.lib.dfr_silu(x)

    def make_instance(self, seed, B, dm, df, scale=1.0):
        x = np.empty((B, dm)); wu = np.empty((dm, df)); wg = np.empty((dm, df))
        wd = np.empty((df, dm))
        self._check(self.lib.dfr_make_instance(seed, B, dm, df, scale, x, wu, wg, wd))
        return x, wu, wg, wd

    def instance(self, x, w_up, w_gate, w_down) -> "RefInstance":
        return RefInstance(self, x, w_up, w_gate, w_down)

    def down_projection(self, a2, w_down):
        B, df = a2.shape
        dm = w_down.shape[1]
        y = np.empty((B, dm))
        self._check(self.lib.dfr_down_projection(np.ascontiguousarray(a2), B, df,
                                                 np.ascontiguousarray(w_down), dm, y))
        return y

    def balanced_ranges(self, extent, parts):
        b = np.zeros(max(parts, 1), dtype=np.int64); e = np.zeros_like(b)
        self._check(self.lib.dfr_balanced_ranges(extent, parts, b, e))
        return list(zip(b.tolist(), e.tolist()))

    def fused_block_bytes(self, B, dm, df, bpe=2):
        return int(self.lib.dfr_fused_block_bytes(B, dm, df, bpe))

    def default_candidate_count(self, B, dm, df):
        return int(self.lib.dfr_default_candidate_count(B, dm, df))


class RefInstance:
    def __init__(self, ref: Reference, x, w_up, w_gate, w_down):
        self.ref = ref
        self.B, self.dm = x.shape
        self.df = w_up.shape[1]
        c = np.ascontiguousarray
        self.h = ref.lib.dfr_instance_create(self.B, self.dm, self.df, c(x), c(w_up),
                                             c(w_gate), c(w_down))
        if not self.h:
            raise ValueError(ref.lib.dfr_last_error().decode())

    def __del__(self):
        if getattr(self, "h", None):
            self.ref.lib.dfr_instance_destroy(self.h)
            self.h = None

    def run_fused(self, tile=None, col_major=True, num_workers=1):
        tm, tn, tk = tile or (self.B, self.df, self.dm)
        y = np.empty((self.B, self.dm))
        self.ref._check(self.ref.lib.dfr_run_fused(self.h, tm, tn, tk, int(col_major),
                                                   num_workers, y))
        return y

    def run_fused_stage1(self, tile=None, col_major=True, num_workers=1):
        tm, tn, tk = tile or (self.B, self.df, self.dm)
        a2 = np.empty((self.B, self.df))
        self.ref._check(self.ref.lib.dfr_run_fused_stage1(self.h, tm, tn, tk,
                                                          int(col_major), num_workers, a2))
        return a2

    def run_variant(self, variant="fused", tile=None, col_major=True):
        tm, tn, tk = tile or (self.B, self.df, self.dm)
        y = np.empty((self.B, self.dm))
        self.ref._check(self.ref.lib.dfr_run_variant(self.h, Reference.VARIANTS[variant],
                                                     tm, tn, tk, int(col_major), y))
        return y

    def oracle_forward(self):
        a2 = np.empty((self.B, self.df)); y = np.empty((self.B, self.dm))
        self.ref._check(self.ref.lib.dfr_oracle_forward(self.h, a2.ctypes.data,
                                                        y.ctypes.data))
        return a2, y

    def run_tp_mlp(self, devices, variant="fused"):
        y = np.empty((self.B, self.dm))
        ev = C.c_int64(); pl = C.c_int64()
        self.ref._check(self.ref.lib.dfr_run_tp_mlp(self.h, devices,
                                                    Reference.VARIANTS[variant], y,
                                                    C.byref(ev), C.byref(pl)))
        return y, ev.value, pl.value
