"""ctypes host layer over the C ABI in include/dfk.h (libdfk.so).

No PyTorch and no CPU fallback: every compute call goes to the sm_100a
kernels in libdfk.so.  If the library is absent it is built in-tree
(nvcc is in the image); if that fails the import raises.
"""
from __future__ import annotations

import ctypes as C
import json
import os
from typing import Optional, Sequence, Tuple

import numpy as np

from . import build as _build

# --- status codes (dfk_status) ---------------------------------------------
OK, ERR_SHAPE, ERR_INVALID, ERR_CUDA, ERR_NCCL, ERR_NOMEM, ERR_UNSUPPORTED, \
    ERR_GATE, ERR_CACHE, ERR_TIMEOUT = range(10)
F64, F32, BF16 = 0, 1, 2
HOST, DEVICE = 0, 1
VARIANT_FUSED, VARIANT_TWO_KERNEL, VARIANT_FOUR_KERNEL = 0, 1, 2
FAMILY_AUTO, FAMILY_TC, FAMILY_GEMV = 0, 1, 2


class DfkError(RuntimeError):
    """Non-shape failure of a dfk call (CUDA, NCCL, gate, cache, ...)."""

    def __init__(self, status: int, msg: str):
        super().__init__(f"[dfk status {status}] {msg}")
        self.status = status


class ShapeError(ValueError):
    """Mirror of deepfusion::ShapeError (a std::invalid_argument)."""

    status = ERR_SHAPE


class InvalidArgument(ValueError):
    status = ERR_INVALID


class GateError(DfkError):
    pass


class CacheError(DfkError):
    pass


class TimeoutError_(DfkError):
    """A fused all-reduce wait on a peer gave up (dfk_context_sync)."""


def library_path() -> str:
    return _build.LIB


def _load() -> C.CDLL:
    override = os.environ.get("DFK_LIB")  # A/B timing of another build (tools/)
    if override:
        return C.CDLL(override)
    path = _build.LIB
    if not os.path.exists(path) or _build._stale():
        try:
            _build.build()
        except Exception as e:  # pragma: no cover - loud failure is the point
            if not os.path.exists(path):
                raise ImportError(
                    f"paper_2602_11808_b200: CUDA library {path} is missing and "
                    f"could not be built ({e}); there is no CPU fallback") from e
    return C.CDLL(path)


lib = _load()


class Config(C.Structure):
    """dfk_config (include/dfk.h): one scheduler candidate / launch config."""

    _fields_ = [("variant", C.c_int32), ("s1_family", C.c_int32),
                ("s1_stages", C.c_int32), ("s1_ctas", C.c_int32),
                ("s1_split_k", C.c_int32), ("down_family", C.c_int32),
                ("down_stages", C.c_int32), ("down_ctas", C.c_int32),
                ("pdl", C.c_int32), ("mutant", C.c_int32),
                ("block_kernel", C.c_int32), ("kbs", C.c_int32),
                ("dynamic_sched", C.c_int32), ("chunk_kb", C.c_int32),
                ("s1_chunk_kb", C.c_int32),
                ("s1_tail", C.c_int32), ("label", C.c_char * 64)]

    @classmethod
    def make(cls, variant=VARIANT_FUSED, s1_family=FAMILY_TC, down_family=FAMILY_TC,
             s1_stages=0, down_stages=0, s1_ctas=0, down_ctas=0, pdl=1, mutant=0,
             s1_split_k=1, block_kernel=0, kbs=0, dynamic_sched=0, chunk_kb=0,
             s1_chunk_kb=0, s1_tail=0, label=""):
        c = cls()
        c.variant, c.s1_family, c.down_family = variant, s1_family, down_family
        c.s1_stages, c.down_stages, c.s1_ctas, c.down_ctas = (s1_stages, down_stages,
                                                              s1_ctas, down_ctas)
        c.pdl, c.mutant, c.s1_split_k = pdl, mutant, s1_split_k
        c.block_kernel, c.kbs = block_kernel, kbs
        c.dynamic_sched, c.chunk_kb = dynamic_sched, chunk_kb
        c.s1_chunk_kb = s1_chunk_kb
        c.s1_tail = s1_tail
        c.label = label.encode()[:63]
        return c

    def as_dict(self) -> dict:
        return {f: getattr(self, f) for f, _ in self._fields_ if f != "label"} | {
            "label": self.label.decode()}

    def __repr__(self) -> str:
        return f"Config({self.as_dict()})"


_vp, _i64, _i32 = C.c_void_p, C.c_int64, C.c_int32
_sigs = {
    "dfk_last_error": ([], C.c_char_p),
    "dfk_version": ([], C.c_char_p),
    "dfk_device_count": ([C.POINTER(C.c_int)], C.c_int),
    "dfk_context_create": ([C.c_int, _vp, C.POINTER(_vp)], C.c_int),
    "dfk_context_destroy": ([_vp], C.c_int),
    "dfk_context_sync": ([_vp], C.c_int),
    "dfk_context_stream": ([_vp, C.POINTER(_vp)], C.c_int),
    "dfk_fingerprint": ([_vp, C.c_char_p, C.c_size_t], C.c_int),
    "dfk_sm_count": ([_vp, C.POINTER(C.c_int)], C.c_int),
    "dfk_weights_create": ([_vp, _vp, _vp, _vp, _i64, _i64, _i32, _i32, _i64, _i64,
                            C.POINTER(_vp)], C.c_int),
    "dfk_weights_destroy": ([_vp], C.c_int),
    "dfk_weights_shape": ([_vp, C.POINTER(_i64), C.POINTER(_i64), C.POINTER(_i64)],
                          C.c_int),
    "dfk_weights_bytes": ([_vp, C.POINTER(_i64)], C.c_int),
    "dfk_stage1": ([_vp, _vp, _vp, _i64, _vp, C.POINTER(Config)], C.c_int),
    "dfk_down": ([_vp, _vp, _vp, _i64, _vp, _i32, C.POINTER(Config)], C.c_int),
    "dfk_forward": ([_vp, _vp, _vp, _i64, _vp, _i32, C.POINTER(Config)], C.c_int),
    "dfk_forward_host": ([_vp, _vp, _vp, _i32, _i64, _vp, _i32, C.POINTER(Config)],
                         C.c_int),
    "dfk_forward_host_async": ([_vp, _vp, _vp, _i64, _vp, C.POINTER(Config)], C.c_int),
    "dfk_candidates": ([_vp, _vp, _i64, C.POINTER(Config), _i32, C.POINTER(_i32)],
                       C.c_int),
    "dfk_candidates_shape": ([_vp, _i64, _i64, _i64, C.POINTER(Config), _i32,
                              C.POINTER(_i32)], C.c_int),
    "dfk_tune": ([_vp, _vp, _i64, C.c_char_p, _i32, _i32, C.POINTER(Config),
                  C.POINTER(_i32), C.c_char_p, C.c_size_t], C.c_int),
    "dfk_select_config": ([_vp, _vp, _i64, C.POINTER(Config)], C.c_int),
    "dfk_cache_lookup": ([C.c_char_p, _i64, _i64, _i64, C.c_char_p, C.c_char_p, C.c_size_t,
                          C.POINTER(C.c_size_t), C.POINTER(_i32)], C.c_int),
    "dfk_cache_store": ([C.c_char_p, C.c_char_p], C.c_int),
    "dfk_tp_unique_id": ([_vp], C.c_int),
    "dfk_tp_init": ([_vp, _vp, C.c_int, C.c_int], C.c_int),
    "dfk_tp_init_all": ([C.POINTER(_vp), C.c_int], C.c_int),
    "dfk_tp_rank": ([_vp, C.POINTER(C.c_int), C.POINTER(C.c_int)], C.c_int),
    "dfk_tp_group_start": ([], C.c_int),
    "dfk_tp_group_end": ([], C.c_int),
    "dfk_tp_forward": ([_vp, _vp, _vp, _i64, _vp, C.POINTER(Config)], C.c_int),
    "dfk_tp_sym_create": ([_vp, _i64, _i64, _vp], C.c_int),
    "dfk_tp_sym_open": ([_vp, _vp, C.c_int, C.c_int], C.c_int),
    "dfk_tp_sym_attach": ([C.POINTER(_vp), C.c_int], C.c_int),
    "dfk_tp_forward_fused": ([_vp, _vp, _vp, _i64, _vp, _i32, C.POINTER(Config)], C.c_int),
    "dfk_profiler_range": ([_vp, C.c_int32], C.c_int),
    "dfk_decode": ([_vp, C.POINTER(_vp), C.c_int32, _vp, _i64, C.c_int32, _vp,
                    C.POINTER(Config), C.c_int32], C.c_int),
    "dfk_balanced_range": ([_i64, _i64, _i64, C.POINTER(_i64), C.POINTER(_i64)],
                           C.c_int),
    "dfk_block_bytes": ([_i64, _i64, _i64, C.POINTER(_i64), C.POINTER(_i64)], C.c_int),
    "dfk_malloc": ([_vp, C.c_size_t, C.POINTER(_vp)], C.c_int),
    "dfk_free": ([_vp, _vp], C.c_int),
    "dfk_host_alloc": ([C.c_size_t, C.POINTER(_vp)], C.c_int),
    "dfk_host_free": ([_vp], C.c_int),
    "dfk_memcpy_h2d": ([_vp, _vp, _vp, C.c_size_t], C.c_int),
    "dfk_memcpy_d2h": ([_vp, _vp, _vp, C.c_size_t], C.c_int),
    "dfk_memset": ([_vp, _vp, C.c_int, C.c_size_t], C.c_int),
    "dfk_host_to_bf16": ([_vp, _i32, C.c_size_t, _vp], C.c_int),
    "dfk_resolve_config": ([_vp, _vp, _i64, _vp, _vp], C.c_int),
    "dfk_host_from_f32": ([_vp, C.c_size_t, _vp, _i32], C.c_int),
    "dfk_host_from_bf16": ([_vp, C.c_size_t, _vp, _i32], C.c_int),
    "dfk_fill_uniform_bf16": ([_vp, _vp, _i64, C.c_uint64, C.c_float, C.c_float],
                              C.c_int),
    "dfk_event_create": ([C.POINTER(_vp)], C.c_int),
    "dfk_event_destroy": ([_vp], C.c_int),
    "dfk_event_record": ([_vp, _vp], C.c_int),
    "dfk_event_elapsed_ms": ([_vp, _vp, C.POINTER(C.c_float)], C.c_int),
    "dfk_flush_l2": ([_vp], C.c_int),
    "dfk_launch_count": ([_vp, C.POINTER(_i64)], C.c_int),
    "dfk_set_trace": ([_vp, _vp, _i64], C.c_int),
}
EXPORTED_SYMBOLS = tuple(_sigs)
for _name, (_args, _res) in _sigs.items():
    if os.environ.get("DFK_LIB") and not hasattr(lib, _name):
        continue  # an older build under A/B test
    _f = getattr(lib, _name)
    _f.argtypes = _args
    _f.restype = _res


def _check(status: int) -> None:
    if status == OK:
        return
    msg = lib.dfk_last_error().decode(errors="replace")
    if status == ERR_SHAPE:
        raise ShapeError(msg)
    if status == ERR_INVALID:
        raise InvalidArgument(msg)
    if status == ERR_GATE:
        raise GateError(status, msg)
    if status == ERR_CACHE:
        raise CacheError(status, msg)
    if status == ERR_TIMEOUT:
        raise TimeoutError_(status, msg)
    raise DfkError(status, msg)


def device_count() -> int:
    n = C.c_int(0)
    _check(lib.dfk_device_count(C.byref(n)))
    return n.value


def balanced_range(extent: int, parts: int, index: int) -> Tuple[int, int]:
    b, e = _i64(), _i64()
    _check(lib.dfk_balanced_range(extent, parts, index, C.byref(b), C.byref(e)))
    return b.value, e.value


def block_bytes(batch: int, d_model: int, d_ff: int) -> Tuple[int, int]:
    """(stage-1, stage-2) algorithmic bytes of one fused block call."""
    s1, s2 = _i64(), _i64()
    _check(lib.dfk_block_bytes(batch, d_model, d_ff, C.byref(s1), C.byref(s2)))
    return s1.value, s2.value


def cache_lookup(path: str, batch: int, d_model: int, d_ff: int,
                 fingerprint: str) -> Optional[dict]:
    """dfk_cache_lookup: the stored ScheduleEntry (a dict) or None on a miss;
    CacheError on a corrupt / other-version file (tuner.hpp:108-113)."""
    need, found = C.c_size_t(0), _i32(0)
    _check(lib.dfk_cache_lookup(path.encode(), batch, d_model, d_ff, fingerprint.encode(),
                                None, 0, C.byref(need), C.byref(found)))
    if not found.value:
        return None
    buf = C.create_string_buffer(need.value)
    _check(lib.dfk_cache_lookup(path.encode(), batch, d_model, d_ff, fingerprint.encode(),
                                buf, need.value, C.byref(need), C.byref(found)))
    return json.loads(buf.value.decode())


def cache_store(path: str, entry: dict) -> None:
    """dfk_cache_store: insert or replace the entry keyed by its shape and
    fingerprint (tuner.hpp:102-106)."""
    _check(lib.dfk_cache_store(path.encode(), json.dumps(entry).encode()))


# --- bf16 helpers (host) ------------------------------------------------------
def to_bf16_bits(a: np.ndarray) -> np.ndarray:
    """fp64/fp32 -> bf16 bits via fp32 with round-to-nearest-even."""
    f = np.ascontiguousarray(a, dtype=np.float32)
    u = f.view(np.uint32).astype(np.uint64)
    nan = np.isnan(f)
    r = ((u + 0x7FFF + ((u >> 16) & 1)) >> 16).astype(np.uint16)
    if nan.any():
        r[nan] = ((u[nan] >> 16) | 0x40).astype(np.uint16)
    return r


def bf16_bits_to_f32(b: np.ndarray) -> np.ndarray:
    return (np.ascontiguousarray(b, dtype=np.uint16).astype(np.uint32) << 16).view(
        np.float32)


_ITEMSIZE = {F64: 8, F32: 4, BF16: 2}


class DeviceArray:
    """A device buffer owned by a Context (row-major, dtype F32 or BF16)."""

    def __init__(self, ctx: "Context", shape: Sequence[int], dtype: int = BF16):
        self.ctx = ctx
        self.shape = tuple(int(s) for s in shape)
        self.dtype = dtype
        self.nbytes = int(np.prod(self.shape)) * _ITEMSIZE[dtype]
        p = _vp()
        _check(lib.dfk_malloc(ctx.h, max(self.nbytes, 16), C.byref(p)))
        self.ptr = p.value

    def __del__(self, _lib=lib):  # (module globals may be gone at exit)
        if getattr(self, "ptr", None) and self.ctx.h:
            _lib.dfk_free(self.ctx.h, self.ptr)
            self.ptr = None

    def upload(self, host: np.ndarray) -> "DeviceArray":
        """Copies a host array in (fp64/fp32 are rounded to bf16 for BF16)."""
        if self.dtype == BF16:
            src = host if host.dtype == np.uint16 else to_bf16_bits(host)
        else:
            src = np.ascontiguousarray(host, dtype=np.float32)
        src = np.ascontiguousarray(src)
        assert src.nbytes == self.nbytes, (src.nbytes, self.nbytes)
        _check(lib.dfk_memcpy_h2d(self.ctx.h, self.ptr, src.ctypes.data, self.nbytes))
        self.ctx.sync()
        return self

    def download(self) -> np.ndarray:
        """Returns the contents as fp32 (bf16 widened exactly)."""
        if self.dtype == BF16:
            out = np.empty(self.shape, dtype=np.uint16)
        else:
            out = np.empty(self.shape, dtype=np.float32)
        self.ctx.sync()
        _check(lib.dfk_memcpy_d2h(self.ctx.h, out.ctypes.data, self.ptr, self.nbytes))
        self.ctx.sync()
        return bf16_bits_to_f32(out) if self.dtype == BF16 else out

    def download_bits(self) -> np.ndarray:
        assert self.dtype == BF16
        out = np.empty(self.shape, dtype=np.uint16)
        self.ctx.sync()
        _check(lib.dfk_memcpy_d2h(self.ctx.h, out.ctypes.data, self.ptr, self.nbytes))
        self.ctx.sync()
        return out

    def fill(self, value_byte: int = 0) -> "DeviceArray":
        _check(lib.dfk_memset(self.ctx.h, self.ptr, value_byte, self.nbytes))
        return self

    def fill_uniform(self, seed: int, lo: float = -1.0, hi: float = 1.0) -> "DeviceArray":
        assert self.dtype == BF16
        _check(lib.dfk_fill_uniform_bf16(self.ctx.h, self.ptr, int(np.prod(self.shape)),
                                         seed, lo, hi))
        return self


class Weights:
    """One block's prepacked weights (dfk_weights_create)."""

    def __init__(self, ctx: "Context", w_gate, w_up, w_down, ff_range=None):
        """w_down None: a stage-1-only set; w_gate and w_up None: a
        down-only set (dfk_weights_create)."""
        self.ctx = ctx
        self.h = None
        present = [a for a in (w_gate, w_up, w_down) if a is not None]
        if not present:
            raise InvalidArgument("no weight matrix given")
        if isinstance(present[0], DeviceArray):
            if w_gate is not None:
                dm, df = w_gate.shape
            else:
                df, dm = w_down.shape
            dtype, mem = present[0].dtype, DEVICE
            ptrs = [a.ptr if a is not None else None for a in (w_gate, w_up, w_down)]
            keep = ()
        else:
            w_gate, w_up, w_down = (np.asarray(a) if a is not None else None
                                    for a in (w_gate, w_up, w_down))
            if w_gate is not None:
                dm, df = w_gate.shape
            else:
                df, dm = w_down.shape
            if ((w_up is not None and w_up.shape != (dm, df)) or
                    (w_gate is not None and w_gate.shape != (dm, df)) or
                    (w_down is not None and w_down.shape != (df, dm))):
                raise ShapeError(
                    f"MlpWeights: w_up {getattr(w_up, 'shape', None)}, w_gate "
                    f"{getattr(w_gate, 'shape', None)}, w_down "
                    f"{getattr(w_down, 'shape', None)} are inconsistent")
            first = next(a for a in (w_gate, w_up, w_down) if a is not None)
            if first.dtype == np.uint16:
                dtype = BF16
            elif first.dtype == np.float32:
                dtype = F32
            else:
                dtype = F64
            npdt = {BF16: np.uint16, F32: np.float32, F64: np.float64}[dtype]
            keep = tuple(np.ascontiguousarray(a, dtype=npdt) if a is not None else None
                         for a in (w_gate, w_up, w_down))
            ptrs = [a.ctypes.data if a is not None else None for a in keep]
            mem = HOST
        f0, f1 = ff_range if ff_range is not None else (0, df)
        h = _vp()
        _check(lib.dfk_weights_create(ctx.h, ptrs[0], ptrs[1], ptrs[2], dm, df, dtype,
                                      mem, f0, f1, C.byref(h)))
        del keep
        self.h = h.value
        self.d_model, self.d_ff_total = int(dm), int(df)
        self.ff_begin, self.d_ff = int(f0), int(f1 - f0)

    def __del__(self, _lib=lib):
        # The context frees every weight set it still owns when it is closed;
        # only destroy explicitly while it is alive.
        if getattr(self, "h", None) and getattr(self.ctx, "h", None):
            _lib.dfk_weights_destroy(self.h)
        self.h = None

    @property
    def packed_bytes(self) -> int:
        b = _i64()
        _check(lib.dfk_weights_bytes(self.h, C.byref(b)))
        return b.value


class Context:
    """A per-GPU execution context (stream, scratch, NCCL comm, schedule)."""

    def __init__(self, device: int = 0, stream: Optional[int] = None):
        h = _vp()
        self.h = None
        _check(lib.dfk_context_create(device, stream, C.byref(h)))
        self.h = h.value
        self.device = device

    def close(self, _lib=lib):
        if getattr(self, "h", None):
            _lib.dfk_context_destroy(self.h)
            self.h = None

    def __del__(self):
        self.close()

    # --- plumbing --------------------------------------------------------
    def sync(self):
        _check(lib.dfk_context_sync(self.h))

    @property
    def stream(self) -> int:
        s = _vp()
        _check(lib.dfk_context_stream(self.h, C.byref(s)))
        return s.value or 0

    @property
    def sm_count(self) -> int:
        n = C.c_int()
        _check(lib.dfk_sm_count(self.h, C.byref(n)))
        return n.value

    def fingerprint(self) -> str:
        buf = C.create_string_buffer(256)
        _check(lib.dfk_fingerprint(self.h, buf, 256))
        return buf.value.decode()

    def resolve_config(self, w: Weights, batch: int, cfg: Optional[Config] = None) -> Config:
        """The configuration a call with `cfg` (None: the scheduler's decision
        or the library default) runs at this batch."""
        out = Config()
        _check(lib.dfk_resolve_config(self.h, w.h, batch, self._cfg(cfg), C.byref(out)))
        return out

    def launch_count(self) -> int:
        n = _i64()
        _check(lib.dfk_launch_count(self.h, C.byref(n)))
        return n.value

    def array(self, shape, dtype=BF16) -> DeviceArray:
        return DeviceArray(self, shape, dtype)

    def weights(self, w_gate, w_up, w_down, ff_range=None) -> Weights:
        return Weights(self, w_gate, w_up, w_down, ff_range)

    def set_trace(self, buf: Optional["DeviceArray"]):
        """Enable (device buffer of uint64 stamps) or disable (None) tracing."""
        if buf is None:
            _check(lib.dfk_set_trace(self.h, None, 0))
        else:
            _check(lib.dfk_set_trace(self.h, buf.ptr, buf.nbytes // 8))

    def flush_l2(self):
        _check(lib.dfk_flush_l2(self.h))

    # --- the hot path ----------------------------------------------------
    @staticmethod
    def _cfg(cfg):
        return C.byref(cfg) if cfg is not None else None

    def stage1(self, w: Weights, x: DeviceArray, a2: DeviceArray, batch: int = None,
               cfg: Optional[Config] = None):
        b = batch or x.shape[0]
        _check(lib.dfk_stage1(self.h, w.h, x.ptr, b, a2.ptr, self._cfg(cfg)))

    def down(self, w: Weights, a2: DeviceArray, y: DeviceArray, batch: int = None,
             cfg: Optional[Config] = None):
        b = batch or a2.shape[0]
        _check(lib.dfk_down(self.h, w.h, a2.ptr, b, y.ptr, y.dtype, self._cfg(cfg)))

    def forward(self, w: Weights, x: DeviceArray, y: DeviceArray, batch: int = None,
                cfg: Optional[Config] = None):
        b = batch or x.shape[0]
        _check(lib.dfk_forward(self.h, w.h, x.ptr, b, y.ptr, y.dtype, self._cfg(cfg)))

    def forward_host(self, w: Weights, x: np.ndarray, cfg: Optional[Config] = None,
                     out_dtype=np.float64) -> np.ndarray:
        """Host-buffer forward (H2D, forward, D2H inside the call)."""
        x = np.ascontiguousarray(x)
        xdt = {np.dtype(np.float64): F64, np.dtype(np.float32): F32,
               np.dtype(np.uint16): BF16}[x.dtype]
        B = x.shape[0]
        y = np.empty((B, w.d_model), dtype=out_dtype)
        ydt = {np.dtype(np.float64): F64, np.dtype(np.float32): F32,
               np.dtype(np.uint16): BF16}[y.dtype]
        _check(lib.dfk_forward_host(self.h, w.h, x.ctypes.data, xdt, B, y.ctypes.data,
                                    ydt, self._cfg(cfg)))
        return y

    def forward_host_into(self, w: Weights, x: np.ndarray, y: np.ndarray,
                          cfg: Optional[Config] = None):
        """forward_host into caller-owned host buffers (x bf16 bits, y fp32)."""
        _check(lib.dfk_forward_host(self.h, w.h, x.ctypes.data, BF16, x.shape[0],
                                    y.ctypes.data, F32, self._cfg(cfg)))

    def forward_host_async(self, w: Weights, x_pinned: np.ndarray, y_pinned: np.ndarray,
                           cfg: Optional[Config] = None):
        """Enqueue H2D(x) + block + D2H(y) on pinned host buffers; no sync."""
        _check(lib.dfk_forward_host_async(self.h, w.h, x_pinned.ctypes.data, x_pinned.shape[0],
                                          y_pinned.ctypes.data, self._cfg(cfg)))

    # --- scheduler -------------------------------------------------------
    def candidates(self, w: Weights, batch: int):
        cap = 64
        arr = (Config * cap)()
        n = _i32()
        _check(lib.dfk_candidates(self.h, w.h, batch, arr, cap, C.byref(n)))
        return [arr[i] for i in range(min(n.value, cap))]

    def tune(self, w: Weights, batch: int, cache_path: Optional[str] = None,
             warmup: int = 1, runs: int = 4):
        """Returns (chosen Config, from_cache, ScheduleEntry dict)."""
        cfg = Config()
        hit = _i32()
        buf = C.create_string_buffer(1 << 16)
        _check(lib.dfk_tune(self.h, w.h, batch,
                            cache_path.encode() if cache_path else None, warmup, runs,
                            C.byref(cfg), C.byref(hit), buf, len(buf)))
        entry = json.loads(buf.value.decode()) if buf.value else {}
        return cfg, bool(hit.value), entry

    def select_config(self, w: Weights, batch: int) -> Config:
        cfg = Config()
        _check(lib.dfk_select_config(self.h, w.h, batch, C.byref(cfg)))
        return cfg

    # --- tensor parallel -------------------------------------------------
    @staticmethod
    def tp_unique_id() -> bytes:
        buf = C.create_string_buffer(128)
        _check(lib.dfk_tp_unique_id(buf))
        return buf.raw

    def tp_init(self, uid: bytes, rank: int, nranks: int):
        buf = C.create_string_buffer(uid, 128)
        _check(lib.dfk_tp_init(self.h, buf, rank, nranks))

    def profiler_range(self, start: bool):
        _check(lib.dfk_profiler_range(self.h, 1 if start else 0))

    def decode(self, layers, x: DeviceArray, steps: int, y: DeviceArray,
               cfg: Optional[Config] = None, graph: bool = True):
        """`steps` passes over `layers`, x <- Y (bf16) after every block
        (time_decode_seconds, bench.cpp:98-115); the last Y lands in y (bf16).
        graph=True captures the sequence into a CUDA graph once and replays it."""
        assert y.dtype == BF16 and x.dtype == BF16
        arr = (_vp * len(layers))(*[w.h for w in layers])
        _check(lib.dfk_decode(self.h, arr, len(layers), x.ptr, x.shape[0], steps, y.ptr,
                              self._cfg(cfg), 1 if graph else 0))

    # --- fused TP all-reduce over NVLink peer memory ---
    def tp_sym_create(self, max_batch: int, d_model: int) -> bytes:
        """Allocate this rank's symmetric workspace; returns its IPC handle."""
        h = (C.c_char * 64)()
        _check(lib.dfk_tp_sym_create(self.h, max_batch, d_model, h))
        return bytes(h)

    def tp_sym_open(self, handles, rank: int, nranks: int):
        """Multi-process: every rank's handle (rank order)."""
        blob = b"".join(handles)
        assert len(blob) == 64 * nranks
        buf = (C.c_char * len(blob)).from_buffer_copy(blob)
        _check(lib.dfk_tp_sym_open(self.h, buf, rank, nranks))

    @staticmethod
    def tp_sym_attach(ctxs):
        """One process driving several contexts (rank i = ctxs[i])."""
        arr = (_vp * len(ctxs))(*[c.h for c in ctxs])
        _check(lib.dfk_tp_sym_attach(arr, len(ctxs)))

    def tp_forward_fused(self, w: Weights, x: DeviceArray, y: DeviceArray,
                         cfg: Optional[Config] = None):
        """This rank's block with the all-reduce inside the kernel; y (F32 or
        BF16) receives the full sum over ranks."""
        _check(lib.dfk_tp_forward_fused(self.h, w.h, x.ptr, x.shape[0], y.ptr, y.dtype,
                                        self._cfg(cfg)))

    def tp_forward(self, w: Weights, x: DeviceArray, y: DeviceArray,
                   cfg: Optional[Config] = None):
        assert y.dtype == F32
        _check(lib.dfk_tp_forward(self.h, w.h, x.ptr, x.shape[0], y.ptr, self._cfg(cfg)))


class Event:
    def __init__(self):
        h = _vp()
        _check(lib.dfk_event_create(C.byref(h)))
        self.h = h.value

    def __del__(self, _lib=lib):
        if getattr(self, "h", None):
            _lib.dfk_event_destroy(self.h)
            self.h = None

    def record(self, ctx: Context):
        _check(lib.dfk_event_record(ctx.h, self.h))

    def elapsed_ms(self, end: "Event") -> float:
        ms = C.c_float()
        _check(lib.dfk_event_elapsed_ms(self.h, end.h, C.byref(ms)))
        return ms.value


class PinnedHost:
    """Page-locked host buffer exposed as a numpy array."""

    def __init__(self, shape, dtype):
        self.arr = None
        n = int(np.prod(shape)) * np.dtype(dtype).itemsize
        p = _vp()
        _check(lib.dfk_host_alloc(n, C.byref(p)))
        self.ptr = p.value
        buf = (C.c_char * n).from_address(self.ptr)
        self.arr = np.frombuffer(buf, dtype=dtype).reshape(shape)

    def __del__(self, _lib=lib):
        if getattr(self, "ptr", None):
            self.arr = None
            _lib.dfk_host_free(self.ptr)
            self.ptr = None
