"""Regional statistics, threshold counts and gradient magnitude (SURVEY §8(a) N2–N5).

Not in the reference (SPEC.md:340 lists regional statistics as a non-goal;
PAPER.md:51,165-168 motivates them).  Definitions, pinned by the oracle
(oracle/hsz_oracle.py: region_stats, region_minmax, threshold_count,
gradient_magnitude):

* regions tile the grid like ``grid.partition`` (origin-aligned, edge regions
  shrunk, row-major region order); the extent is clipped to the grid;
* per region exact S1 = sum(q), S2 = sum(q^2) (int128), qmin, qmax;
  mean_r = S1/size*2eps, var_r = (size*S2 - S1^2)/(size(size-1))*(2eps)^2
  (NaN below two points); min_r = qmin*2eps, max_r = qmax*2eps;
* threshold count = #regions with min_r < tau <= max_r;
* gradient magnitude = eps*sqrt(sum_k D_k^2) with D_k the integer central
  differences of fields._axis_central_diff.

One K-REG pass computes every per-region integer; one small kernel
finalises the floats and the count.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np

from .._nvtx import ranged
from .. import _lib, device as devmod
from ..compressors import CompressedStream
from ..stages import Stage, _check_stage, count_stage_work


@dataclass(frozen=True)
class RegionStats:
    region: tuple
    grid: tuple          # regions per axis
    s1: np.ndarray       # int64
    s2_lo: np.ndarray    # uint64 low / int64 high halves of the exact int128 S2 (see .s2)
    s2_hi: np.ndarray
    qmin: np.ndarray     # int32
    qmax: np.ndarray     # int32
    size: np.ndarray     # int64
    mean: np.ndarray     # float64
    var: np.ndarray      # float64
    vmin: np.ndarray     # float64 = qmin * 2eps
    vmax: np.ndarray     # float64 = qmax * 2eps
    threshold: float | None = None
    crossing_count: int | None = None

    @property
    def s2(self) -> np.ndarray:
        """Exact S2 per region: int64 when every value fits, else Python ints (object)."""
        hi = self.s2_hi.astype(np.int64)
        lo = self.s2_lo.astype(np.uint64)
        if not hi.any() and (lo < np.uint64(1 << 63)).all():
            return lo.astype(np.int64).reshape(self.grid)
        vals = [(int(h) << 64) | int(l) for h, l in zip(hi.ravel(), lo.ravel())]
        return np.array(vals, dtype=object).reshape(self.grid)


def _region_tuple(region, nd):
    return (int(region),) * nd if np.isscalar(region) else tuple(int(r) for r in region)


def region_reduce_device(q_dev, eps: float, region, tau: float = float("nan")):
    """Device-side per-region reduction + finalisation; returns CUDA tensors (views of one buffer,
    ``buf``, which the host reads in a single copy)."""
    nd = q_dev.dim()
    reg = _region_tuple(region, nd)
    grid, buf, v = devmod.region_reduce(q_dev, reg)
    nr = v["s1"].numel()
    _lib.call("hszg_region_finalize", _lib.ptr(v["s1"]), _lib.ptr(v["s2lo"]), _lib.ptr(v["s2hi"]),
              _lib.ptr(v["qmin"]), _lib.ptr(v["qmax"]), _lib.ptr(v["size"]), nr, 2.0 * eps, float(tau),
              _lib.ptr(v["mean"]), _lib.ptr(v["var"]), _lib.ptr(v["vmin"]), _lib.ptr(v["vmax"]), _lib.ptr(v["count"]),
              _lib.stream_handle())
    return dict(grid=grid, region=tuple(min(r, n) for r, n in zip(reg, q_dev.shape)), buf=buf, **v)


def _region_device(c: CompressedStream, stage: Stage, region, tau: float):
    """Per-region outputs on the device: fused from the bytes for the block-mean kinds when the regions
    align with the blocks (hszg_region_stream, K-REG), else over the reconstructed q."""
    stage = Stage(stage)
    if stage not in (Stage.DECORRELATED, Stage.QUANTIZED):
        raise ValueError("regional statistics run on stage 2 or 3 integers")
    _check_stage(c, stage)
    count_stage_work(c, stage)
    if c.kind.is_block_mean:
        d = c.device().validate()
        nd = len(c.shape.dims)
        reg = _region_tuple(region, nd)
        dims = tuple(int(n) for n in c.shape.dims)
        regc = tuple(min(r, n) for r, n in zip(reg, dims))
        grid = tuple(-(-n // r) for n, r in zip(dims, regc))
        nr = int(np.prod(grid))
        buf = devmod.region_buffer(nr)
        v = devmod.region_views(buf, nr)
        ws = _lib.workspace(64 * nr)
        err = _lib.Err()
        reg_arr = (ctypes.c_int64 * 3)(*(list(reg) + [1] * (3 - nd)))
        st = _lib.lib().hszg_region_stream(ctypes.byref(d.geom), ctypes.byref(d.desc),
                                            ctypes.cast(reg_arr, ctypes.c_void_p), _lib.ptr(v["s1"]),
                                            _lib.ptr(v["s2lo"]), _lib.ptr(v["s2hi"]), _lib.ptr(v["qmin"]),
                                            _lib.ptr(v["qmax"]), _lib.ptr(v["size"]), _lib.ptr(ws), ws.numel(),
                                            _lib.stream_handle(), ctypes.byref(err))
        if st == _lib.OK:
            return _finalize(dict(grid=grid, region=regc, buf=buf, **v), c.eps, tau)
        if st != _lib.UNSUPPORTED_STAGE:
            _lib.raise_for(st, err, "hszg_region_stream")
    t = _lib.torch()
    q = c.device().reconstruct(t.int32)
    return region_reduce_device(q, c.eps, region, tau)


def _finalize(r, eps: float, tau: float):
    v = r
    nr = v["s1"].numel()
    _lib.call("hszg_region_finalize", _lib.ptr(v["s1"]), _lib.ptr(v["s2lo"]), _lib.ptr(v["s2hi"]),
              _lib.ptr(v["qmin"]), _lib.ptr(v["qmax"]), _lib.ptr(v["size"]), nr, 2.0 * eps, float(tau),
              _lib.ptr(v["mean"]), _lib.ptr(v["var"]), _lib.ptr(v["vmin"]), _lib.ptr(v["vmax"]), _lib.ptr(v["count"]),
              _lib.stream_handle())
    return r


def _quantized(c: CompressedStream, stage: Stage):
    stage = Stage(stage)
    if stage not in (Stage.DECORRELATED, Stage.QUANTIZED):
        raise ValueError("regional statistics run on stage 2 or 3 integers")
    _check_stage(c, stage)
    count_stage_work(c, stage)
    t = _lib.torch()
    return c.device().reconstruct(t.int32)


@ranged("hsz/region_stats")
def region_stats(c: CompressedStream, region, stage: Stage = Stage.QUANTIZED,
                 tau: float | None = None) -> RegionStats:
    """Per-region mean/variance/min/max (N2, N3) and optionally the tau crossing count (N4)."""
    r = _region_device(c, stage, region, float("nan") if tau is None else tau)
    g = r["grid"]
    nr = int(np.prod(g))
    host = r["buf"].cpu().numpy()                 # every output in one device -> host copy
    w = [host[k * nr:(k + 1) * nr] for k in range(devmod.REGION_WORDS)]
    mm = w[8].view(np.int32)
    return RegionStats(
        region=r["region"], grid=g,
        s1=w[0].reshape(g), s2_lo=w[1].view(np.uint64).reshape(g), s2_hi=w[2].reshape(g),
        qmin=mm[:nr].reshape(g), qmax=mm[nr:].reshape(g), size=w[3].reshape(g),
        mean=w[4].view(np.float64).reshape(g), var=w[5].view(np.float64).reshape(g),
        vmin=w[6].view(np.float64).reshape(g), vmax=w[7].view(np.float64).reshape(g),
        threshold=tau, crossing_count=None if tau is None else int(host[devmod.REGION_WORDS * nr]),
    )


def region_minmax(c: CompressedStream, region, stage: Stage = Stage.QUANTIZED):
    """N3: (qmin, qmax, min_r, max_r) arrays shaped like the region grid."""
    s = region_stats(c, region, stage)
    return s.qmin, s.qmax, s.vmin, s.vmax


@ranged("hsz/threshold_count")
def threshold_count(c: CompressedStream, region, tau: float, stage: Stage = Stage.QUANTIZED) -> int:
    """N4: number of regions with min_r < tau <= max_r (only the count leaves the device)."""
    return int(_region_device(c, stage, region, float(tau))["count"].item())


def gradient_magnitude(c: CompressedStream, stage: Stage = Stage.QUANTIZED, out: str = "numpy", out_dtype=None):
    """N5: eps * sqrt(sum_k D_k^2) on the integer central differences."""
    from .fields import compute_field_op

    return compute_field_op(c, "gradient_magnitude", stage, out, out_dtype).components[0]
