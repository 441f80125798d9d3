"""Finite-difference operators on intermediate representations (reference hsz/analytics/fields.py).

Unit grid spacing; the 1/2 of the central difference is absorbed into the
2*eps dequantization scale, so integer stencils are scaled by eps
(derivatives) or 2*eps (Laplacian); outputs are exactly 0 wherever a
neighbour would leave the domain.  All stencils run in the K-STEN kernel
(``hszg_stencil``) on int32 indices reconstructed on the device; the
stage-4 variants reproduce the reference's float64 rounding sequence
operation by operation, and the stage-2 variants (nd kinds) are
bit-identical to stage 3 by construction — the same integers
(fields.py:108-168 proves the identity; test_fields.py:39-48 checks it).

Axis convention: the x derivative differentiates along axis 0 (slowest).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .._nvtx import ranged
from .. import _lib, device as devmod
from ..compressors import CompressedStream, CompressorKind, DecorrelatedStream, _as_device, recorrelate
from ..errors import UnsupportedStageError
from ..quant import QuantizedField
from ..stages import Stage, _check_stage, count_stage_work, sliding_window

AXIS_NAMES = ("dx", "dy", "dz")


@dataclass(frozen=True)
class DerivedField:
    op: str
    components: tuple
    component_names: tuple


def _host(outs, out):
    if out == "torch":
        return tuple(outs)
    return tuple(o.cpu().numpy() for o in outs)


def _q_dev(values):
    t = _lib.torch()
    return _as_device(values, t.int32)


def _dtype(out_dtype):
    t = _lib.torch()
    if out_dtype is None:
        return t.float64
    return {np.dtype(np.float32): t.float32, np.dtype(np.float64): t.float64}.get(np.dtype(out_dtype), out_dtype) \
        if not isinstance(out_dtype, t.dtype) else out_dtype


# ---------------------------------------------------------------------------
# Quantized-index (stage 3) and float (stage 4) paths


def derivative_from_dq(q: QuantizedField, out: str = "numpy", out_dtype=None) -> DerivedField:
    """(q[i+1]-q[i-1]) * eps per axis (fields.py:67-72)."""
    qd = _q_dev(q.values)
    outs = devmod.stencil(_lib.OP_DERIV, [qd], [q.eps], False, _dtype(out_dtype))
    return DerivedField("derivative", _host(outs, out), AXIS_NAMES[: qd.dim()])


def laplacian_from_dq(q: QuantizedField, out: str = "numpy", out_dtype=None) -> DerivedField:
    """(sum of neighbours - 2*nd*q) * 2eps (fields.py:75-80)."""
    qd = _q_dev(q.values)
    if qd.dim() < 2:
        raise ValueError("Laplacian requires 2D or 3D data")
    outs = devmod.stencil(_lib.OP_LAPLACIAN, [qd], [q.eps], False, _dtype(out_dtype))
    return DerivedField("laplacian", _host(outs, out), ("lap",))


def _f_dev(field):
    t = _lib.torch()
    if isinstance(field, t.Tensor):
        return field.to(_lib.device()).to(t.float64).contiguous()
    return _as_device(np.asarray(field, dtype=np.float64), t.float64)


def derivative_from_df(field, out: str = "numpy", out_dtype=None) -> DerivedField:
    """(d[i+1]-d[i-1])/2 in float64 (fields.py:83-86)."""
    fd = _f_dev(field)
    outs = devmod.stencil(_lib.OP_DERIV, [fd], [1.0], 2, _dtype(out_dtype))
    return DerivedField("derivative", _host(outs, out), AXIS_NAMES[: fd.dim()])


def laplacian_from_df(field, out: str = "numpy", out_dtype=None) -> DerivedField:
    """fields.py:89-93."""
    fd = _f_dev(field)
    if fd.dim() < 2:
        raise ValueError("Laplacian requires 2D or 3D data")
    outs = devmod.stencil(_lib.OP_LAPLACIAN, [fd], [1.0], 2, _dtype(out_dtype))
    return DerivedField("laplacian", _host(outs, out), ("lap",))


# ---------------------------------------------------------------------------
# Decorrelated (stage 2) paths, multidimensional kinds only


def _require_nd_stream(stream: DecorrelatedStream):
    if not stream.kind.is_nd:
        raise UnsupportedStageError(
            f"{stream.kind.cli_name} does not support stencil operations on "
            "decorrelated data (no multidimensional layout)"
        )


def derivative_from_dp(stream: DecorrelatedStream, out: str = "numpy", out_dtype=None) -> DerivedField:
    """fields.py:108-136 — identical integers to the stage-3 stencil."""
    _require_nd_stream(stream)
    return derivative_from_dq(recorrelate(stream), out, out_dtype)


def laplacian_from_dp(stream: DecorrelatedStream, out: str = "numpy", out_dtype=None) -> DerivedField:
    """fields.py:139-168."""
    _require_nd_stream(stream)
    return laplacian_from_dq(recorrelate(stream), out, out_dtype)


# ---------------------------------------------------------------------------
# Stage dispatch straight from a compressed stream


def _stage_q(c: CompressedStream, stage: Stage):
    if stage in (Stage.META,):
        raise UnsupportedStageError("stencil operations need stage >= decorrelated")
    _check_stage(c, stage)
    if stage == Stage.DECORRELATED and not c.kind.is_nd:
        raise UnsupportedStageError(
            f"{c.kind.cli_name} does not support stencil operations on "
            "decorrelated data (no multidimensional layout)"
        )
    t = _lib.torch()
    q = c.device().reconstruct(t.int32)
    count_stage_work(c, stage)
    return q


_OPS = {"derivative": _lib.OP_DERIV, "laplacian": _lib.OP_LAPLACIAN, "gradient_magnitude": _lib.OP_GRADMAG}
_FAST_QLIM = 1 << 27        # int32 stencils (table emitter) are exact while |q| < 2^27 (stencil.cuh)
_SMS = 148


def _fused_layers(dims) -> int:
    """Block layers per CTA of hszg_fused_blocks for a whole field: fewest (CTA waves x (layers per CTA + one
    layer of pipeline fill)) on one CTA per SM (512^3: 8 layers, 1024 CTAs; tools/probe_fused_modes.py measured
    8 < 64 < 4 < 16 layers)."""
    n0, n1, n2 = dims
    xy = -(-(n2 // 8) // 16) * -(-(n1 // 8) // 2)
    nlay = n0 // 8
    best = None
    for zl in range(1, nlay + 1):
        cost = -(-(xy * -(-nlay // zl)) // _SMS) * (zl + 1)
        if best is None or cost < best[0]:
            best = (cost, zl)
    return best[1]


def _fused_stencil(c: CompressedStream, op: str, dtype):
    """HSZX_ND (8^3 blocks, 3-D) derivative / Laplacian with fp32 outputs in one pass from the compressed
    bytes (hszg_fused_blocks with only the requested outputs: q never reaches HBM), bit-identical to
    reconstruct + K-STEN: fl32 of the reference float64 by the table emitter while |q| < 2^27 (bounded here
    by the block means and the bit width), else the fp64-conversion emitter.  None when not eligible."""
    t = _lib.torch()
    dims = tuple(c.shape.dims)
    if (dtype != t.float32 or c.kind != CompressorKind.HSZX_ND or len(dims) != 3 or tuple(c.block_dims) != (8, 8, 8)
            or any(n % 8 for n in dims) or op not in ("derivative", "laplacian")):
        return None
    ds = c.device().validate()
    if not ds.desc.canonical or ds.desc.max_bitwidth > 16:
        return None
    qmax = ds.mean_absmax() + (1 << ds.desc.max_bitwidth)
    mode = 2 if (qmax < _FAST_QLIM and 2.0 ** -125 <= float(c.eps) <= 2.0 ** 90) else 1
    outs = [t.empty(dims, dtype=t.float32, device=_lib.device()) for _ in range(3 if op == "derivative" else 1)]
    ptrs = [_lib.ptr(o) for o in outs] + [None] if op == "derivative" else [None, None, None, _lib.ptr(outs[0])]
    import ctypes
    err = _lib.Err()
    _lib.call("hszg_fused_blocks", ctypes.byref(ds.geom), ctypes.byref(ds.desc), 0, dims[0], None, None,
              (ctypes.c_void_p * 4)(*ptrs), None, _fused_layers(dims), mode, _lib.stream_handle(),
              ctypes.byref(err), err=err)
    return outs

@ranged("hsz/compute_field_op")
def compute_field_op(c: CompressedStream, op: str, stage: Stage, out: str = "numpy", out_dtype=None) -> DerivedField:
    """Derivative / Laplacian (and gradient magnitude, N5) of one compressed field (fields.py:181-196)."""
    stage = Stage(stage)
    if op not in _OPS:
        if stage == Stage.META:
            raise UnsupportedStageError("stencil operations need stage >= decorrelated")
        raise ValueError(f"unknown field operation {op!r}")
    outs = None
    if stage in (Stage.DECORRELATED, Stage.QUANTIZED):
        _check_stage(c, stage)
        outs = _fused_stencil(c, op, _dtype(out_dtype))
    if outs is not None:
        count_stage_work(c, stage)
        ndim = 3
    else:
        q = _stage_q(c, stage)
        ndim = q.dim()
        if op == "laplacian" and q.dim() < 2:
            raise ValueError("Laplacian requires 2D or 3D data")
        outs = devmod.stencil(_OPS[op], [q], [c.eps], stage == Stage.FULL, _dtype(out_dtype))
    if op == "derivative":
        return DerivedField("derivative", _host(outs, out), AXIS_NAMES[:ndim])
    if op == "laplacian":
        return DerivedField("laplacian", _host(outs, out), ("lap",))
    return DerivedField("gradient_magnitude", _host(outs, out), ("gradmag",))


def _check_components(sources):
    shapes = {c.shape.dims for c in sources}
    if len(shapes) != 1:
        raise ValueError(f"component shapes differ: {sorted(shapes)}")
    kinds = {c.kind for c in sources}
    if len(kinds) != 1:
        raise ValueError("all components must use the same compressor")
    ndims = len(next(iter(shapes)))
    if ndims != len(sources):
        raise ValueError(f"{ndims}D vector field needs {ndims} components, got {len(sources)}")


def _vector_op(sources, stage, opcode, name, names, out, out_dtype):
    stage = Stage(stage)
    _check_components(sources)
    qs = [_stage_q(c, stage) for c in sources]
    outs = devmod.stencil(opcode, qs, [c.eps for c in sources], stage == Stage.FULL, _dtype(out_dtype))
    return DerivedField(name, _host(outs, out), names[: len(outs)])


@ranged("hsz/divergence")
def divergence(sources, stage: Stage, out: str = "numpy", out_dtype=None) -> DerivedField:
    """sum_k D_k(u_k) in float64 in component order (fields.py:216-222), one fused launch."""
    return _vector_op(sources, stage, _lib.OP_DIVERGENCE, "divergence", ("div",), out, out_dtype)


@ranged("hsz/curl")
def curl(sources, stage: Stage, out: str = "numpy", out_dtype=None) -> DerivedField:
    """2-D scalar curl dy(u)-dx(v); 3-D right-handed curl (fields.py:225-236)."""
    names = ("curl",) if len(sources) == 2 else ("cx", "cy", "cz")
    return _vector_op(sources, stage, _lib.OP_CURL, "curl", names, out, out_dtype)


# ---------------------------------------------------------------------------
# Out-of-core streaming (Algorithm 3)


@ranged("hsz/streamed_derivative")
def streamed_derivative(c: CompressedStream, out: str = "numpy", out_dtype=None, from_host=None) -> DerivedField:
    """Slab-streamed derivative holding at most three quantized slabs (fields.py:243-272).

    Each window (prev[-1], cur, nxt[:1]) is assembled on the device and run
    through the same stencil kernel; bit-identical to derivative_from_dq.
    """
    if not c.kind.is_nd:
        raise UnsupportedStageError("streamed derivative needs an nd compressor")
    t = _lib.torch()
    dims = c.shape.dims
    dtype = _dtype(out_dtype)
    # out="numpy": the components are filled slab by slab in host memory (with from_host, nothing
    # field-sized ever lives on the device: the out-of-core use of Algorithm 3)
    on_host = out != "torch"
    if on_host:
        comps = [np.zeros(dims, dtype=np.float32 if dtype == t.float32 else np.float64) for _ in dims]
    else:
        comps = [t.zeros(dims, dtype=dtype, device=_lib.device()) for _ in dims]
    row = 0
    for _, prev, cur, nxt in sliding_window(c, Stage.QUANTIZED, out="torch", from_host=from_host):
        rows = cur.shape[0]
        parts = [cur]
        top = 0
        if prev is not None:
            parts.insert(0, prev[-1:])
            top = 1
        if nxt is not None:
            parts.append(nxt[:1])
        ext = t.empty((sum(p.shape[0] for p in parts),) + tuple(dims[1:]), dtype=t.int32, device=_lib.device())
        r0 = 0
        for p in parts:
            ext[r0:r0 + p.shape[0]].copy_(p)
            r0 += p.shape[0]
        outs = devmod.stencil(_lib.OP_DERIV, [ext], [c.eps], False, dtype)
        for ax in range(len(dims)):
            if on_host:
                comps[ax][row:row + rows] = outs[ax][top:top + rows].cpu().numpy()
            else:
                comps[ax][row:row + rows].copy_(outs[ax][top:top + rows])
        row += rows
    return DerivedField("derivative", tuple(comps) if on_host else _host(comps, out), AXIS_NAMES[: len(dims)])
