"""Mirror of the reference's C++ operator API over the B200 C ABI.

Same names, argument meaning and error classes as
``/root/reference/proj/include/deepfusion/{tensor,swiglu,fused,tp,tuner}.hpp``
so code (and tests) written against the reference read the same here.
Matrices are numpy fp64 row-major arrays (the reference ``Matrix``,
tensor.hpp:73-128); every call converts them to bf16, runs the sm_100a
kernels through libdfk.so and widens the result back to fp64.  There is no
CPU compute path.

Differences that follow from the hardware, documented rather than hidden:

* ``TileConfig`` is validated exactly like the reference (dims >= 1,
  fused.cpp:16-22) but is a *hint*: the GPU tile (64 A2 columns x full
  d_model per CTA pass) is fixed by the tensor-core shape and the launch
  parameters come from the profile-driven scheduler.  Results are
  tile-independent within tolerance, as the reference's tiling-invariance
  criterion requires (verification.cpp:278-308).
* ``num_workers`` is accepted and ignored: the CTA grid is the parallelism.
* Results match the fp64 reference within the bf16 tolerance (max relative
  error <= 1e-2 on Y), not bit-exactly.
"""
from __future__ import annotations

import enum
from dataclasses import dataclass, field
from typing import Dict, List, Optional

import numpy as np

from . import runtime as rt
from .runtime import ShapeError

__all__ = [
    "ShapeError", "LoopOrder", "VariantTag", "TileConfig", "KernelConfig", "MlpShape",
    "MlpWeights", "make_random_weights", "run_fused_stage1", "run_fused",
    "down_projection", "run_stage1", "run_variant", "run_four_kernel", "run_two_kernel",
    "ColRange", "ShardPlan", "ShardScheme", "balanced_ranges", "make_plan", "run_tp_mlp",
    "CollectiveKind", "CollectiveEvent", "CollectiveLog", "TpResult", "comm_volume_bytes",
    "CommModel", "Tuner", "default_fingerprint", "silu", "sigmoid", "context",
]


class LoopOrder(enum.Enum):
    RowMajorTiling = 0
    ColumnMajorTiling = 1


class VariantTag(enum.Enum):
    FourKernel = 0
    TwoKernel = 1
    Fused = 2


_VARIANT_TO_ABI = {VariantTag.Fused: rt.VARIANT_FUSED,
                   VariantTag.TwoKernel: rt.VARIANT_TWO_KERNEL,
                   VariantTag.FourKernel: rt.VARIANT_FOUR_KERNEL}


@dataclass
class TileConfig:
    tile_m: int = 1
    tile_n: int = 1
    tile_k: int = 1
    loop_order: LoopOrder = LoopOrder.ColumnMajorTiling

    def validate(self) -> None:  # fused.cpp:16-22
        if self.tile_m < 1 or self.tile_n < 1 or self.tile_k < 1:
            raise ShapeError(f"TileConfig: tile dimensions must be >= 1, got "
                             f"{self.describe()}")

    def clamped(self, shape: "MlpShape") -> "TileConfig":  # fused.cpp:24-30
        return TileConfig(min(self.tile_m, shape.batch), min(self.tile_n, shape.d_ff),
                          min(self.tile_k, shape.d_model), self.loop_order)

    def describe(self) -> str:  # fused.cpp:32-37
        o = "row" if self.loop_order == LoopOrder.RowMajorTiling else "col"
        return f"m{self.tile_m}_n{self.tile_n}_k{self.tile_k}_{o}"


@dataclass
class KernelConfig:
    variant: VariantTag = VariantTag.Fused
    tile: TileConfig = field(default_factory=TileConfig)
    label: str = ""
    gpu: Optional[rt.Config] = None  # explicit launch config (None = scheduler)


@dataclass
class MlpShape:
    batch: int = 1
    d_model: int = 1
    d_ff: int = 1

    def validate(self) -> None:  # tensor.cpp:83-89
        if self.batch < 1 or self.d_model < 1 or self.d_ff < 1:
            raise ShapeError(f"MlpShape: all dimensions must be >= 1, got {self}")

    def ff_ratio_typical(self) -> bool:  # tensor.cpp:91-95
        r = self.d_ff / self.d_model
        return 3.5 <= r <= 4.0


@dataclass(eq=False)
class MlpWeights:
    w_up: np.ndarray
    w_gate: np.ndarray
    w_down: np.ndarray
    shape: MlpShape

    def validate(self) -> None:  # swiglu.cpp:26-39
        self.shape.validate()
        s = self.shape
        for name, m, exp in (("w_up", self.w_up, (s.d_model, s.d_ff)),
                             ("w_gate", self.w_gate, (s.d_model, s.d_ff)),
                             ("w_down", self.w_down, (s.d_ff, s.d_model))):
            if tuple(m.shape) != exp:
                raise ShapeError(f"MlpWeights: {name} is {m.shape[0]}x{m.shape[1]}, "
                                 f"expected {exp[0]}x{exp[1]}")


def sigmoid(x: float) -> float:  # tensor.hpp:155-161
    if x >= 0.0:
        return 1.0 / (1.0 + np.exp(-x))
    e = np.exp(x)
    return e / (1.0 + e)


def silu(x: float) -> float:
    return x * sigmoid(x)


def make_random_weights(shape: MlpShape, seed: int, scale: float = 1.0) -> MlpWeights:
    """Seeded U[-scale, scale) weights (device-independent numpy generator)."""
    shape.validate()
    g = np.random.default_rng(seed)
    return MlpWeights(g.uniform(-scale, scale, (shape.d_model, shape.d_ff)),
                      g.uniform(-scale, scale, (shape.d_model, shape.d_ff)),
                      g.uniform(-scale, scale, (shape.d_ff, shape.d_model)), shape)


# --- device state -------------------------------------------------------------
_CTX: Optional[rt.Context] = None
_HANDLES: Dict[tuple, rt.Weights] = {}


def context() -> rt.Context:
    global _CTX
    if _CTX is None:
        _CTX = rt.Context(0)
    return _CTX


def _key(*arrs) -> tuple:
    return tuple((a.__array_interface__["data"][0], a.shape) for a in arrs)


def _register(w_gate, w_up, w_down, ff_range=None) -> rt.Weights:
    k = _key(w_gate, w_up, w_down) + (ff_range,)
    h = _HANDLES.get(k)
    if h is None:
        if len(_HANDLES) > 16:
            _HANDLES.clear()
        h = context().weights(w_gate, w_up, w_down, ff_range)
        _HANDLES[k] = h
    return h


def _gpu_cfg(config: Optional[KernelConfig]) -> Optional[rt.Config]:
    if config is None:
        return None
    if config.gpu is not None:
        c = rt.Config.from_buffer_copy(config.gpu)
        c.variant = _VARIANT_TO_ABI[config.variant]
        return c
    if config.variant == VariantTag.Fused:
        return None  # scheduler's pick for the fused layout
    return rt.Config.make(variant=_VARIANT_TO_ABI[config.variant])


def _f64(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float64)


# --- operators ----------------------------------------------------------------
def run_fused_stage1(x, w_up, w_gate, tile: TileConfig, a2: np.ndarray,
                     num_workers: int = 1, cfg: Optional[rt.Config] = None) -> None:
    """A2 = (X W_up) * silu(X W_gate) into the caller-preallocated a2
    (fused.hpp:61-63; validation fused.cpp:49-68)."""
    tile.validate()
    x, w_up, w_gate = _f64(x), _f64(w_up), _f64(w_gate)
    if (w_up.shape[0] != x.shape[1] or w_gate.shape[0] != x.shape[1]
            or w_up.shape[1] != w_gate.shape[1]):
        raise ShapeError(f"run_fused_stage1: inconsistent dims, x is {x.shape}, "
                         f"w_up is {w_up.shape}, w_gate is {w_gate.shape}")
    if a2.shape != (x.shape[0], w_up.shape[1]):
        raise ShapeError(f"run_fused_stage1: a2 is {a2.shape}, expected "
                         f"{(x.shape[0], w_up.shape[1])}")
    B, dm = x.shape
    df = w_up.shape[1]
    zeros = np.zeros((df, dm))
    h = _register(w_gate, w_up, zeros)
    ctx = context()
    xd = ctx.array((B, dm)).upload(x)
    ad = ctx.array((B, df))
    ctx.stage1(h, xd, ad, cfg=cfg)
    a2[...] = ad.download()


def run_fused(x, w: MlpWeights, tile: TileConfig = None, num_workers: int = 1,
              cfg: Optional[rt.Config] = None) -> np.ndarray:
    """Fused stage 1 then down (fused.cpp:209-216), host buffers in and out."""
    w.validate()
    (tile or TileConfig()).validate()
    x = _f64(x)
    if x.shape[1] != w.shape.d_model:
        raise ShapeError(f"executor: x has {x.shape[1]} columns, weights expect "
                         f"d_model={w.shape.d_model}")
    h = _register(_f64(w.w_gate), _f64(w.w_up), _f64(w.w_down))
    return context().forward_host(h, x, cfg=cfg)


def down_projection(a2, w_down) -> np.ndarray:
    """Y = A2 W_down (swiglu.cpp:214-226)."""
    a2, w_down = _f64(a2), _f64(w_down)
    if a2.shape[1] != w_down.shape[0]:
        raise ShapeError(f"down_projection: a2 has {a2.shape[1]} columns, w_down has "
                         f"{w_down.shape[0]} rows")
    B, df = a2.shape
    dm = w_down.shape[1]
    zeros = np.zeros((dm, df))
    h = _register(zeros, zeros, w_down)
    ctx = context()
    ad = ctx.array((B, df)).upload(a2)
    yd = ctx.array((B, dm), rt.F32)
    ctx.down(h, ad, yd)
    return yd.download().astype(np.float64)


def run_stage1(variant: VariantTag, x, w: MlpWeights, a2: np.ndarray,
               tile: TileConfig = None) -> None:
    """Dispatch stage 1 by variant (fused.cpp:241-256)."""
    if not isinstance(variant, VariantTag):
        raise rt.InvalidArgument("run_stage1: unknown variant")
    w.validate()
    if variant == VariantTag.Fused:
        run_fused_stage1(x, w.w_up, w.w_gate, tile or TileConfig(), a2)
        return
    x = _f64(x)
    B = x.shape[0]
    h = _register(_f64(w.w_gate), _f64(w.w_up), _f64(w.w_down))
    ctx = context()
    xd = ctx.array((B, w.shape.d_model)).upload(x)
    ad = ctx.array((B, w.shape.d_ff))
    ctx.stage1(h, xd, ad, cfg=rt.Config.make(variant=_VARIANT_TO_ABI[variant]))
    a2[...] = ad.download()


def run_variant(config: KernelConfig, x, w: MlpWeights) -> np.ndarray:
    """Full block under a kernel config (fused.cpp:258-264)."""
    w.validate()
    config.tile.validate()
    return run_fused(x, w, config.tile, cfg=_gpu_cfg(config))


def run_four_kernel(x, w: MlpWeights) -> np.ndarray:
    return run_variant(KernelConfig(VariantTag.FourKernel), x, w)


def run_two_kernel(x, w: MlpWeights) -> np.ndarray:
    return run_variant(KernelConfig(VariantTag.TwoKernel), x, w)


# --- tensor parallelism (tp.hpp) -----------------------------------------------
@dataclass(frozen=True)
class ColRange:
    begin: int = 0
    end: int = 0

    def size(self) -> int:
        return self.end - self.begin


class ShardScheme(enum.Enum):
    CompoundSingleAllReduce = 0
    NaivePerGemmAllGather = 1


class CollectiveKind(enum.Enum):
    AllReduce = 0
    AllGather = 1


@dataclass
class CollectiveEvent:
    kind: CollectiveKind
    payload_elements_per_device: int


@dataclass
class CollectiveLog:
    events: List[CollectiveEvent] = field(default_factory=list)


@dataclass
class ShardPlan:
    num_devices: int = 1
    ff_ranges: List[ColRange] = field(default_factory=list)
    scheme: ShardScheme = ShardScheme.CompoundSingleAllReduce

    def validate(self, d_ff: int) -> None:  # tp.cpp:31-53
        if self.num_devices < 1 or len(self.ff_ranges) != self.num_devices:
            raise ShapeError("ShardPlan: range count does not match num_devices")
        cursor = 0
        for r in self.ff_ranges:
            if r.begin != cursor or r.size() < 1:
                raise ShapeError("ShardPlan: ranges must be contiguous, disjoint and "
                                 f"non-empty; offending range [{r.begin}, {r.end}) at "
                                 f"cursor {cursor}")
            cursor = r.end
        if cursor != d_ff:
            raise ShapeError(f"ShardPlan: ranges cover [0, {cursor}) but d_ff is {d_ff}")


@dataclass
class TpResult:
    output: np.ndarray
    log: CollectiveLog
    stage1_shards: List[np.ndarray]


def balanced_ranges(extent: int, parts: int) -> List[ColRange]:
    """tp.cpp:8-29 through the C ABI (dfk_balanced_range)."""
    return [ColRange(*rt.balanced_range(extent, parts, i)) for i in range(parts)] \
        if parts >= 1 else [ColRange(*rt.balanced_range(extent, parts, 0))]


def make_plan(d_ff: int, num_devices: int,
              scheme: ShardScheme = ShardScheme.CompoundSingleAllReduce) -> ShardPlan:
    return ShardPlan(num_devices, balanced_ranges(d_ff, num_devices), scheme)


def run_tp_mlp(x, w: MlpWeights, plan: ShardPlan, executor: KernelConfig) -> TpResult:
    """Compound TP block (tp.cpp:140-167).

    Each shard's weights are prepacked once (dfk_weights_create with the
    shard's [ff_begin, ff_end)); the shard runs stage 1 and the down
    projection into an fp32 partial Y on the GPU.  With one process the
    partials are summed in device-index order (the reference's
    simulated_all_reduce, tp.cpp:90-105); the multi-GPU path with a real
    ncclAllReduce is ``Context.tp_forward`` (one rank per GPU).
    """
    w.validate()
    plan.validate(w.shape.d_ff)
    if plan.scheme != ShardScheme.CompoundSingleAllReduce:
        raise rt.InvalidArgument("run_tp_mlp: plan scheme must be "
                                 "CompoundSingleAllReduce")
    x = _f64(x)
    if x.shape[1] != w.shape.d_model:
        raise ShapeError("run_tp_mlp: x column count does not match d_model")
    ctx = context()
    B = x.shape[0]
    xd = ctx.array((B, w.shape.d_model)).upload(x)
    partials, shards = [], []
    cfg = _gpu_cfg(executor)
    for r in plan.ff_ranges:
        h = _register(_f64(w.w_gate), _f64(w.w_up), _f64(w.w_down), (r.begin, r.end))
        ad = ctx.array((B, r.size()))
        yd = ctx.array((B, w.shape.d_model), rt.F32)
        ctx.stage1(h, xd, ad, cfg=cfg)
        ctx.down(h, ad, yd, cfg=cfg)
        shards.append(ad.download().astype(np.float64))
        partials.append(yd.download().astype(np.float64))
    out = partials[0].copy()
    for p in partials[1:]:
        out += p
    log = CollectiveLog([CollectiveEvent(CollectiveKind.AllReduce, B * w.shape.d_model)])
    return TpResult(out, log, shards)


class CommModel(enum.Enum):
    Logical = 0
    Ring = 1


def comm_volume_bytes(log: CollectiveLog, num_devices: int, model: CommModel,
                      bytes_per_element: int = 2) -> float:
    """tp.cpp:237-261."""
    if num_devices < 1:
        raise ShapeError("comm_volume_bytes: num_devices must be >= 1")
    p = float(num_devices)
    total = 0.0
    for ev in log.events:
        payload = float(ev.payload_elements_per_device * bytes_per_element)
        if model == CommModel.Logical:
            total += payload
        elif ev.kind == CollectiveKind.AllReduce:
            total += 2.0 * (p - 1.0) / p * payload
        else:
            total += (p - 1.0) / p * payload
    return total


# --- scheduler (tuner.hpp) -----------------------------------------------------
def default_fingerprint() -> str:
    return context().fingerprint()


class Tuner:
    """Front door of the profile-driven scheduler (tuner.hpp:117-137):
    cache lookup, else profile + select + store (dfk_tune)."""

    def __init__(self, cache_path: str = "", warmup: int = 1, runs: int = 4):
        self.cache_path = cache_path
        self.warmup, self.runs = warmup, runs
        self.profile_invocations = 0
        self.last_was_cache_hit = False

    def get_or_tune(self, w: MlpWeights, batch: int) -> dict:
        w.validate()
        h = _register(_f64(w.w_gate), _f64(w.w_up), _f64(w.w_down))
        cfg, hit, entry = context().tune(h, batch, self.cache_path or None,
                                         self.warmup, self.runs)
        self.last_was_cache_hit = hit
        if not hit:
            self.profile_invocations += 1
        entry["chosen_gpu_config"] = cfg
        return entry
