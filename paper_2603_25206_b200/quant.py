"""Linear-scaling quantization under an absolute error bound (reference hsz/quant.py).

q = floor(d * (1/(2*eps)) + 0.5) in float64 with the multiply and the add
rounded separately (quant.py:73-76), dequantized as q * (2*eps).  Both run on
the GPU (``hszg_quantize_*`` / the stage-4 epilogue of ``hszg_reconstruct``);
this module keeps the reference's host API on top.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np

from . import _lib
from .errors import ZeroValueRangeError
from .grid import GridShape

QMAX = 2**31 - 2


@dataclass(frozen=True)
class ErrorBound:
    """User-requested error bound, absolute or value-range relative (quant.py:23-41)."""

    mode: str
    requested: float

    def __post_init__(self):
        if self.mode not in ("abs", "rel"):
            raise ValueError(f"error bound mode must be abs or rel, got {self.mode!r}")
        if not self.requested > 0:
            raise ValueError(f"error bound must be positive, got {self.requested}")

    @classmethod
    def parse(cls, text: str) -> "ErrorBound":
        mode, _, value = text.partition(":")
        if not value:
            raise ValueError(f"error bound must look like abs:0.1, got {text!r}")
        return cls(mode, float(value))


@dataclass(frozen=True)
class QuantizedField:
    """Grid of int32 quantization indices plus the resolved eps (quant.py:44-53).

    ``values`` is a numpy array for the drop-in API or a CUDA tensor in
    device mode (``out="torch"``).
    """

    values: object
    eps: float

    @property
    def shape(self) -> GridShape:
        return GridShape(tuple(self.values.shape))


def to_device(x, dtype=None):
    """Host array -> CUDA tensor (no copy if already on the device)."""
    t = _lib.torch()
    if isinstance(x, t.Tensor):
        out = x if x.is_cuda else x.to(_lib.device(), non_blocking=False)
        return out if dtype is None else out.to(dtype)
    arr = np.ascontiguousarray(x)
    return t.from_numpy(arr).to(_lib.device())


def field_minmax(field_dev):
    """(min, max, nonfinite count) of a float field, computed on the GPU."""
    t = _lib.torch()
    n = field_dev.numel()
    out = t.zeros(3, dtype=t.float64, device=_lib.device())
    bad = t.zeros(1, dtype=t.int64, device=_lib.device())
    ws = _lib.workspace(148 * 8 * 32 + 256)
    fn = "hszg_minmax_f32" if field_dev.dtype == t.float32 else "hszg_minmax_f64"
    _lib.call(fn, _lib.ptr(field_dev), n, _lib.ptr(out), _lib.ptr(bad), _lib.ptr(ws), ws.numel(),
              _lib.stream_handle())
    mm = out.cpu().numpy()
    return float(mm[0]), float(mm[1]), int(bad.item())


def _float_field(values):
    t = _lib.torch()
    d = to_device(values)
    if d.dtype not in (t.float32, t.float64):
        d = d.to(t.float64)
    return d.contiguous()


def resolve_eps(field, bound: ErrorBound) -> float:
    """Resolve a bound to an absolute eps (quant.py:56-66); the value range comes from the GPU."""
    if bound.mode == "abs":
        return float(bound.requested)
    lo, hi, _ = field_minmax(_float_field(field).reshape(-1))
    if hi == lo:
        raise ZeroValueRangeError("constant field has zero value range; use an absolute error bound")
    return float(bound.requested) * (hi - lo)


def quantize_device(field_dev, eps: float):
    """CUDA float tensor -> CUDA int32 tensor of indices (quant.py:69-82)."""
    t = _lib.torch()
    if not eps > 0:
        raise ValueError(f"eps must be positive, got {eps}")
    recip = 1.0 / (2.0 * eps)
    flat = field_dev.reshape(-1)
    q = t.empty(flat.numel(), dtype=t.int32, device=_lib.device())
    err = _lib.Err()
    ws = _lib.workspace(256)
    fn = "hszg_quantize_f32" if flat.dtype == t.float32 else "hszg_quantize_f64"
    _lib.call(fn, _lib.ptr(flat), flat.numel(), recip, _lib.ptr(q), _lib.ptr(ws), ws.numel(), _lib.stream_handle(),
              ctypes.byref(err), err=err)
    return q.reshape(field_dev.shape)


def quantize(values, eps: float):
    """Quantize floats to int32 indices; scalar inputs give a 0-d array (quant.py:69-82)."""
    if not eps > 0:
        raise ValueError(f"eps must be positive, got {eps}")
    arr = np.asarray(values)
    d = _float_field(arr.reshape(-1) if arr.ndim else arr.reshape(1))
    q = quantize_device(d, eps).cpu().numpy()
    return q.reshape(arr.shape)


def dequantize(q, eps: float):
    """Recover floats as q * (2*eps) in float64 (quant.py:85-87), on the GPU."""
    t = _lib.torch()
    arr = np.asarray(q)
    qd = to_device(arr.astype(np.int32, copy=False).reshape(-1) if arr.ndim else arr.astype(np.int32).reshape(1))
    out = dequantize_device(qd, eps)
    return out.cpu().numpy().reshape(arr.shape)


def dequantize_device(q_dev, eps: float, dtype=None):
    """int32 CUDA tensor -> float CUDA tensor, q * (2*eps) rounded once (stages.py:88)."""
    t = _lib.torch()
    dtype = dtype or t.float64
    flat = q_dev.reshape(-1).to(t.int32).contiguous()
    out = t.empty(flat.numel(), dtype=dtype, device=_lib.device())
    code = _lib.F64 if dtype == t.float64 else _lib.F32
    _lib.call("hszg_dequantize", _lib.ptr(flat), flat.numel(), 2.0 * eps, _lib.ptr(out), code, _lib.stream_handle())
    return out.reshape(q_dev.shape)


def quantize_field(field, eps: float) -> QuantizedField:
    """quant.py:90-93."""
    d = _float_field(np.asarray(field) if not _is_tensor(field) else field)
    _, _, bad = field_minmax(d.reshape(-1))
    if bad:
        raise ValueError("field contains NaN or Inf; refusing to quantize")
    return QuantizedField(quantize_device(d, eps).cpu().numpy(), float(eps))


def _is_tensor(x):
    try:
        import torch

        return isinstance(x, torch.Tensor)
    except ImportError:  # pragma: no cover
        return False
