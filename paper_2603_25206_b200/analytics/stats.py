"""Mean, standard deviation and variance on intermediate representations
(reference hsz/analytics/stats.py).

The integer sums are computed exactly on the GPU (int128 accumulators,
``hszg_reduce_*``) — fused straight from the compressed bytes wherever the
stage allows it (① metadata, ② weighted residual sums / block-mean sums,
③ sums of q for the HSZx family need no scatter) — and finished on the
host with the reference's own Python-int expressions, so every scalar is
bit-identical to the reference.  ``var`` is added next to
``mean`` / ``std``.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

from .._nvtx import ranged
from .. import _lib, device as devmod
from ..compressors import CompressedStream, CompressorKind, DecorrelatedStream, _as_device, _stored_block_dims
from ..errors import UnsupportedStageError
from ..quant import QuantizedField
from ..stages import Stage, _check_stage, count_stage_work

# hszg_reduce_stream modes
MODE_HSZP_WEIGHTED = 1
MODE_LORENZO_WEIGHTED = 2
MODE_BLOCK_MEAN_Q = 3
MODE_META = 4
NO_EXTREMA = 0x100          # HSZG_REDUCE_NO_EXTREMA: min / max not computed (leaner decode)


@dataclass(frozen=True)
class StatResult:
    value: float
    stage_used: Stage
    op: str


def _int32_device(values):
    t = _lib.torch()
    if isinstance(values, t.Tensor):
        return values.reshape(-1).to(t.int32).contiguous()
    arr = np.asarray(values).reshape(-1)
    a64 = arr.astype(np.int64, copy=False)
    if a64.size and (a64.min() < -(2**31) or a64.max() > 2**31 - 1):
        raise ValueError("exact integer reductions take int32-range values")
    return _as_device(a64.astype(np.int32), t.int32)


def _exact_sum(values) -> int:
    """Exact integer sum (stats.py:30-39), int128 on the GPU."""
    v = _int32_device(values)
    if v.numel() == 0:
        return 0
    return _lib.read_sums(devmod.reduce_i32(v)).s1


def _exact_dot(a, b) -> int:
    """Exact integer dot product (stats.py:42-55), int128 on the GPU."""
    a = _int32_device(a)
    b = _int32_device(b)
    if a.numel() == 0:
        return 0
    return _lib.read_sums(devmod.reduce_dot(a, b)).s1


def _std_from_sums(s1: int, s2: int, n: int, eps: float) -> float:
    """stats.py:58-62."""
    if n < 2:
        raise ValueError("standard deviation requires at least 2 points")
    num = s2 * n - s1 * s1
    return math.sqrt(num / (n * (n - 1))) * 2.0 * eps


def _var_from_sums(s1: int, s2: int, n: int, eps: float) -> float:
    """N1: the radicand of _std_from_sums scaled by (2*eps)^2."""
    if n < 2:
        raise ValueError("variance requires at least 2 points")
    num = s2 * n - s1 * s1
    return num / (n * (n - 1)) * ((2.0 * eps) * (2.0 * eps))


def _block_mean_moments(s1: int, s2: int, weighted: int, n: int):
    """HSZx stage-2 integer mean mu = (2W+n)//(2n) and sum((q-mu)^2) (stats.py:130-136).

    sum((p + M_b - mu)^2) = sum(q^2) - 2 mu sum(q) + n mu^2 exactly, with q = p + M_b.
    """
    mu = (2 * weighted + n) // (2 * n)
    return mu, s2 - 2 * mu * s1 + n * mu * mu


# ---------------------------------------------------------------------------
# Mean


def mean_from_meta(metadata, block_sizes, eps: float) -> float:
    """Mean from per-block integer means: sum(M_b*S_b)/N * 2eps (stats.py:69-77)."""
    metadata = np.asarray(metadata)
    if metadata.size == 0:
        raise ValueError("no block metadata")
    n = int(np.asarray(block_sizes, dtype=np.int64).sum())
    return _exact_dot(metadata, block_sizes) / n * (2.0 * eps)


def _stream_sums(stream: DecorrelatedStream, mode: int):
    g = _lib.make_geom(int(stream.kind), stream.shape.dims,
                       _stored_block_dims(stream.kind, stream.shape, stream.geometry), stream.eps)
    p = _int32_device(stream.values)
    meta = _int32_device(stream.metadata) if stream.metadata is not None else None
    return _lib.read_sums(devmod.reduce_array(g, p, meta, mode))


def _weighted_mode(kind: CompressorKind) -> int:
    if kind.is_block_mean:
        return MODE_BLOCK_MEAN_Q
    return MODE_HSZP_WEIGHTED if kind == CompressorKind.HSZP else MODE_LORENZO_WEIGHTED


def mean_from_dp(stream: DecorrelatedStream) -> float:
    """Mean from decorrelated values without reconstructing indices (stats.py:80-92)."""
    n = stream.shape.total
    total = _stream_sums(stream, _weighted_mode(stream.kind)).s1
    return total / n * (2.0 * float(stream.eps))


def _lorenzo_weighted_sum(p, dims) -> int:
    """sum(q) from Lorenzo residuals via separable weights (stats.py:95-112), on the GPU."""
    dims = tuple(int(d) for d in dims)
    g = _lib.make_geom(int(CompressorKind.HSZP_ND), dims, dims, 1.0)
    return _lib.read_sums(devmod.reduce_array(g, _int32_device(p), None, MODE_LORENZO_WEIGHTED)).s1


def mean_from_dq(q: QuantizedField) -> float:
    """(sum(q)/N) * 2eps (stats.py:115-118)."""
    v = _int32_device(q.values)
    total = _lib.read_sums(devmod.reduce_i32(v)).s1
    return total / v.numel() * (2.0 * q.eps)


# ---------------------------------------------------------------------------
# Standard deviation / variance


def _q_sums_from_stream(stream: DecorrelatedStream):
    """Exact (sum q, sum q^2) for a decorrelated stream: block-mean kinds fused, prefix kinds via q."""
    if stream.kind.is_block_mean:
        return _stream_sums(stream, MODE_BLOCK_MEAN_Q)
    from ..compressors import recorrelate

    t = _lib.torch()
    ds = DecorrelatedStream(_int32_device(stream.values), None, stream.geometry, stream.shape, stream.eps,
                            stream.kind)
    q = recorrelate(ds).values
    return _lib.read_sums(devmod.reduce_i32(q))


def std_from_dp(stream: DecorrelatedStream) -> float:
    """Standard deviation from decorrelated values (stats.py:125-144)."""
    n = stream.shape.total
    eps = float(stream.eps)
    sums = _q_sums_from_stream(stream)
    if stream.kind.is_block_mean:
        if n < 2:
            raise ValueError("standard deviation requires at least 2 points")
        weighted = _exact_dot(stream.metadata, stream.geometry.block_sizes())
        _, dd = _block_mean_moments(sums.s1, sums.s2, weighted, n)
        return math.sqrt(dd / (n - 1)) * 2.0 * eps
    return _std_from_sums(sums.s1, sums.s2, n, eps)


def _lorenzo_prefix_std(p, dims, eps: float) -> float:
    """Algorithm 4 (stats.py:147-165): exact sums of the reconstructed q."""
    dims = tuple(int(d) for d in dims)
    from ..compressors import recorrelate
    from ..grid import GridShape, partition

    shape = GridShape(dims)
    ds = DecorrelatedStream(_int32_device(p), None, partition(shape, dims), shape, eps, CompressorKind.HSZP_ND)
    q = recorrelate(ds).values
    s = _lib.read_sums(devmod.reduce_i32(q))
    return _std_from_sums(s.s1, s.s2, shape.total, eps)


def std_from_dq(q: QuantizedField) -> float:
    """stats.py:168-173."""
    v = _int32_device(q.values)
    s = _lib.read_sums(devmod.reduce_i32(v))
    return _std_from_sums(s.s1, s.s2, v.numel(), q.eps)


def var_from_dq(q: QuantizedField) -> float:
    v = _int32_device(q.values)
    s = _lib.read_sums(devmod.reduce_i32(v))
    return _var_from_sums(s.s1, s.s2, v.numel(), q.eps)


def _float_moments(x_dev):
    """(mean, sum of squared deviations) of a float64 CUDA array, two passes (stats.py:176-186)."""
    t = _lib.torch()
    x = x_dev.reshape(-1).to(t.float64).contiguous()
    ws = _lib.workspace(devmod.REDUCE_WS)
    out = _lib.sums_tensor()
    _lib.call("hszg_reduce_flt", _lib.ptr(x), x.numel(), None, _lib.ptr(out), _lib.ptr(ws), ws.numel(),
              _lib.stream_handle())
    mean = _lib.read_sums(out).f1 / x.numel()
    mean_dev = t.tensor([mean], dtype=t.float64, device=_lib.device())
    _lib.call("hszg_reduce_flt", _lib.ptr(x), x.numel(), _lib.ptr(mean_dev), _lib.ptr(out), _lib.ptr(ws), ws.numel(),
              _lib.stream_handle())
    return mean, _lib.read_sums(out).f2


def mean_from_df(field) -> float:
    x = _as_device(np.asarray(field, dtype=np.float64) if not _is_t(field) else field)
    return _float_moments(x)[0]


def std_from_df(field) -> float:
    x = _as_device(np.asarray(field, dtype=np.float64) if not _is_t(field) else field)
    if x.numel() < 2:
        raise ValueError("standard deviation requires at least 2 points")
    _, m2 = _float_moments(x)
    return math.sqrt(m2 / (x.numel() - 1))


def _is_t(x):
    t = _lib.torch()
    return isinstance(x, t.Tensor)


def eps_of(stream: DecorrelatedStream) -> float:
    return float(stream.eps)


# ---------------------------------------------------------------------------
# Stage dispatch: fused device paths straight from the compressed stream


def _stage4_moments(d, eps, n):
    """Float-domain moments of fl(q*2eps) without materialising the floats (two fused passes)."""
    t = _lib.torch()
    q = d.reconstruct(t.int32)
    s = _lib.read_sums(devmod.reduce_f64(q, 2.0 * eps))
    mean = s.f1 / n
    mean_dev = t.tensor([mean], dtype=t.float64, device=_lib.device())
    s2 = _lib.read_sums(devmod.reduce_f64(q, 2.0 * eps, mean_dev))
    return mean, s2.f2


def stream_sums(c: CompressedStream, stage: Stage):
    """Exact device sums for (c, stage) as used by compute_stat; also the multi-GPU partials."""
    t = _lib.torch()
    d = c.device()
    if stage == Stage.META:
        return _lib.read_sums(d.reduce(MODE_META))
    if c.kind.is_block_mean:
        return _lib.read_sums(d.reduce(MODE_BLOCK_MEAN_Q | NO_EXTREMA))
    fused = d.quantized_sums()          # q reduced where it is formed, never written (HSZP, 3-D HSZP_ND)
    if fused is not None:
        return _lib.read_sums(fused)
    q = d.reconstruct(t.int32)
    return _lib.read_sums(devmod.reduce_i32(q))


@ranged("hsz/compute_stat")
def compute_stat(c: CompressedStream, op: str, stage: Stage) -> StatResult:
    """Run mean / std / var at the given stage of a compressed stream (stats.py:195-212)."""
    stage = Stage(stage)
    if op not in ("mean", "std", "var"):
        raise ValueError(f"unknown statistic {op!r}")
    if op != "mean" and stage == Stage.META:
        raise UnsupportedStageError("standard deviation needs stage >= decorrelated")
    _check_stage(c, stage)
    d = c.device()
    n = c.shape.total
    eps = c.eps
    count_stage_work(c, stage)
    if stage == Stage.META:
        total = _lib.read_sums(d.reduce(MODE_META)).s1
        return StatResult(total / n * (2.0 * eps), stage, op)
    if stage == Stage.FULL:
        mean, m2 = _stage4_moments(d, eps, n)
        if op == "mean":
            return StatResult(mean, stage, op)
        if n < 2:
            raise ValueError("standard deviation requires at least 2 points")
        var = m2 / (n - 1)
        return StatResult(math.sqrt(var) if op == "std" else var, stage, op)
    if op == "mean":
        # sum q is the same exact integer at stages 2 and 3: the weighted residual sum (prefix kinds,
        # stats.py:88/95-112) or the block-mean sum (HSZX*) straight from the bytes — no reconstruction
        total = _lib.read_sums(d.reduce(_weighted_mode(c.kind) | NO_EXTREMA)).s1
        return StatResult(total / n * (2.0 * eps), stage, op)
    s = stream_sums(c, stage)
    if stage == Stage.DECORRELATED and c.kind.is_block_mean:
        if n < 2:
            raise ValueError("standard deviation requires at least 2 points")
        weighted = _lib.read_sums(d.reduce(MODE_META)).s1
        _, dd = _block_mean_moments(s.s1, s.s2, weighted, n)
        if op == "std":
            return StatResult(math.sqrt(dd / (n - 1)) * 2.0 * eps, stage, op)
        return StatResult(dd / (n - 1) * ((2.0 * eps) * (2.0 * eps)), stage, op)
    fn = _std_from_sums if op == "std" else _var_from_sums
    return StatResult(fn(s.s1, s.s2, n, eps), stage, op)
