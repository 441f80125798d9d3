"""The four HSZ pipelines and their decorrelation primitives (reference hsz/compressors.py).

HSZP / HSZX treat the field as a flat 1-D array; HSZP_ND / HSZX_ND keep the
multidimensional layout.  The HSZp family predicts from previous neighbours
(1-D previous value, nd Lorenzo corner sum), the HSZx family subtracts a
truncated integer block mean stored as per-block metadata.

Every per-element transform (quantize, decorrelate, chunk encode,
recorrelate, permutations) runs on the GPU through libhszg.so; this module
keeps the reference's classes and signatures and the host-side geometry.
A ``CompressedStream`` produced by :func:`compress` is born on the device
(its host ``payload`` / ``chunk_offsets`` / ``metadata`` are fetched lazily),
and one read from bytes is uploaded once on first use.
"""

from __future__ import annotations

import ctypes
import os
import enum
from dataclasses import dataclass, field
from functools import cached_property

import numpy as np

from ._nvtx import ranged
from . import _lib, codec
from .device import DeviceStream
from .errors import EpsTooSmallError, MissingContextError
from .grid import BlockGeometry, GridShape, canonical_order, partition
from .quant import ErrorBound, QuantizedField, _float_field, field_minmax, quantize_device, resolve_eps

_PMAX = 2**31 - 1

DEFAULT_BLOCK_1D = 32
DEFAULT_BLOCK_ND = {2: (8, 8), 3: (8, 8, 8)}


class CompressorKind(enum.IntEnum):
    HSZP = 0
    HSZP_ND = 1
    HSZX = 2
    HSZX_ND = 3

    @property
    def is_nd(self) -> bool:
        return self in (CompressorKind.HSZP_ND, CompressorKind.HSZX_ND)

    @property
    def is_block_mean(self) -> bool:
        return self in (CompressorKind.HSZX, CompressorKind.HSZX_ND)

    @property
    def cli_name(self) -> str:
        return self.name.lower().replace("_nd", "-nd")

    @classmethod
    def from_name(cls, name: str) -> "CompressorKind":
        key = name.strip().lower().replace("-", "_")
        try:
            return cls[key.upper()]
        except KeyError:
            raise ValueError(f"unknown compressor {name!r}") from None


def _to_host(x):
    if x is None:
        return None
    t = _lib.torch()
    if isinstance(x, t.Tensor):
        return x.cpu().numpy()
    return x


def _as_device(x, dtype=None):
    t = _lib.torch()
    if isinstance(x, t.Tensor):
        d = x if x.is_cuda else x.to(_lib.device())
    else:
        d = t.from_numpy(np.ascontiguousarray(x)).to(_lib.device())
    if dtype is not None and d.dtype != dtype:
        d = d.to(dtype)
    return d.contiguous()


@dataclass
class DecorrelatedStream:
    """Decorrelated integers in canonical stream order plus block metadata (compressors.py:57-84)."""

    values: object            # int32, stream order (numpy, or CUDA tensor in device mode)
    metadata: object          # int32 block means (HSZx family) or None
    geometry: BlockGeometry
    shape: GridShape
    eps: float
    kind: CompressorKind
    source: DeviceStream | None = field(default=None, repr=False, compare=False)

    def _geom(self):
        return _lib.make_geom(int(self.kind), self.shape.dims, _stored_block_dims(self.kind, self.shape,
                                                                                self.geometry), self.eps)

    def as_grid(self):
        """Residuals rearranged to row-major grid layout (hszg_scatter_grid)."""
        t = _lib.torch()
        g = self._geom()
        vals = _as_device(self.values, t.int32).reshape(-1)
        out = t.empty(self.shape.total, dtype=t.int32, device=_lib.device())
        _lib.call("hszg_scatter_grid", ctypes.byref(g), _lib.ptr(vals), None, 0, _lib.ptr(out), _lib.stream_handle())
        out = out.reshape(self.shape.dims)
        return out if isinstance(self.values, t.Tensor) else out.cpu().numpy()

    def metadata_grid(self):
        """Per-point block mean expanded to grid layout (int64, hszg_metadata_grid)."""
        if self.metadata is None:
            raise ValueError("stream has no block-mean metadata")
        t = _lib.torch()
        g = self._geom()
        meta = _as_device(self.metadata, t.int32)
        out = t.empty(self.shape.total, dtype=t.int64, device=_lib.device())
        _lib.call("hszg_metadata_grid", ctypes.byref(g), _lib.ptr(meta), _lib.ptr(out), _lib.stream_handle())
        out = out.reshape(self.shape.dims)
        return out if isinstance(self.values, t.Tensor) else out.cpu().numpy()


def _stored_block_dims(kind, shape: GridShape, geometry: BlockGeometry):
    """Per-original-axis block dims as stored in the container (S,1,...) for flat kinds."""
    if kind.is_nd:
        return tuple(geometry.block_dims)
    return (int(geometry.block_dims[0]),) + (1,) * (shape.ndims - 1)


def effective_geometry(kind: CompressorKind, shape: GridShape, block_dims) -> BlockGeometry:
    """Blocking used for streaming: flattened for 1-D kinds (compressors.py:87-93)."""
    if kind.is_nd:
        return partition(shape, block_dims)
    return partition(shape.flattened(), (block_dims[0],))


def stream_perm(kind: CompressorKind, shape: GridShape, geometry: BlockGeometry) -> np.ndarray:
    """Stream position -> flat row-major index (compressors.py:96-102)."""
    if kind == CompressorKind.HSZX_ND:
        return canonical_order(shape, geometry, "block-contiguous")
    return canonical_order(shape, geometry, "global-row-major")


def segment_bounds(kind: CompressorKind, shape: GridShape, geometry: BlockGeometry) -> list:
    """Stream segments at which chunks restart (compressors.py:105-119)."""
    if kind == CompressorKind.HSZP_ND:
        slab = int(np.prod(shape.dims[1:], dtype=np.int64))
        return [(i * slab, (i + 1) * slab) for i in range(shape.dims[0])]
    sizes = geometry.block_sizes()
    ends = np.cumsum(sizes)
    starts = ends - sizes
    return list(zip(starts.tolist(), ends.tolist()))


def block_int_mean(values) -> int:
    """Integer block mean truncated toward zero (compressors.py:122-131)."""
    values = np.asarray(values, dtype=np.int64)
    if values.size == 0:
        raise ValueError("empty block")
    total = int(values.sum())
    mean, rem = divmod(total, values.size)
    if total < 0 and rem != 0:
        mean += 1
    return int(mean)


def _decorrelate_device(q_dev, kind: CompressorKind, shape: GridShape, block_dims, eps: float):
    """GPU decorrelation -> (p stream tensor, metadata tensor or None, geom)."""
    t = _lib.torch()
    g = _lib.make_geom(int(kind), shape.dims, block_dims, eps)
    p = t.empty(shape.total, dtype=t.int32, device=_lib.device())
    meta = t.empty(max(int(g.n_blocks), 1), dtype=t.int32, device=_lib.device()) if kind.is_block_mean else None
    err = _lib.Err()
    ws = _lib.workspace(256)
    q = _as_device(q_dev, t.int32).reshape(-1)
    _lib.call("hszg_decorrelate", ctypes.byref(g), _lib.ptr(q), _lib.ptr(p), _lib.ptr(meta) if meta is not None else None,
              _lib.ptr(ws), ws.numel(), _lib.stream_handle(), ctypes.byref(err), err=err)
    if meta is not None:
        meta = meta[: int(g.n_blocks)]
    return p, meta, g


def _wrap_ds(p, meta, geometry, shape, eps, kind, device_mode=False):
    if not device_mode:
        p = _to_host(p)
        meta = _to_host(meta)
    return DecorrelatedStream(p, meta, geometry, shape, eps, kind)


def decorrelate_hszp(q: QuantizedField) -> DecorrelatedStream:
    """Previous-value prediction over the flattened array (compressors.py:149-157)."""
    shape = q.shape
    bd = (min(DEFAULT_BLOCK_1D, shape.total),) + (1,) * (shape.ndims - 1)
    p, _, _ = _decorrelate_device(q.values, CompressorKind.HSZP, shape, bd, q.eps)
    geometry = partition(shape.flattened(), (bd[0],))
    return _wrap_ds(p, None, geometry, shape, q.eps, CompressorKind.HSZP, _is_dev(q.values))


def decorrelate_lorenzo_nd(q: QuantizedField) -> DecorrelatedStream:
    """Multidimensional Lorenzo residuals, zero padding (compressors.py:160-176)."""
    shape = q.shape
    if shape.ndims < 2:
        raise ValueError("Lorenzo decorrelation requires 2D or 3D data")
    bd = _clip_block_dims(DEFAULT_BLOCK_ND[shape.ndims], shape)
    p, _, _ = _decorrelate_device(q.values, CompressorKind.HSZP_ND, shape, bd, q.eps)
    return _wrap_ds(p, None, partition(shape, bd), shape, q.eps, CompressorKind.HSZP_ND, _is_dev(q.values))


def decorrelate_hszx(q: QuantizedField, geometry: BlockGeometry, kind: CompressorKind) -> DecorrelatedStream:
    """Subtract the truncated integer block mean in every block (compressors.py:179-198)."""
    shape = q.shape
    bd = _stored_block_dims(kind, shape, geometry)
    p, meta, _ = _decorrelate_device(q.values, kind, shape, bd, q.eps)
    return _wrap_ds(p, meta, geometry, shape, q.eps, kind, _is_dev(q.values))


def decorrelate(q: QuantizedField, kind: CompressorKind, geometry: BlockGeometry):
    """compressors.py:229-238."""
    if kind == CompressorKind.HSZP:
        ds = decorrelate_hszp(q)
    elif kind == CompressorKind.HSZP_ND:
        ds = decorrelate_lorenzo_nd(q)
    else:
        return decorrelate_hszx(q, geometry, kind)
    ds.geometry = geometry
    return ds


def recorrelate(stream: DecorrelatedStream, out_dtype=None) -> QuantizedField:
    """Exact integer inverse of the decorrelation (compressors.py:201-226), on the GPU."""
    t = _lib.torch()
    shape = stream.shape
    n_vals = stream.values.numel() if isinstance(stream.values, t.Tensor) else np.asarray(stream.values).size
    if n_vals != shape.total:
        if stream.kind.is_block_mean:
            raise ValueError("stream length does not match grid size")
        raise MissingContextError("partial prefix-predicted stream; predecessor context required")
    g = _lib.make_geom(int(stream.kind), shape.dims, _stored_block_dims(stream.kind, shape, stream.geometry),
                       stream.eps)
    p = _as_device(stream.values, t.int32).reshape(-1)
    meta = _as_device(stream.metadata, t.int32) if stream.metadata is not None else None
    out = t.empty(shape.dims, dtype=t.int32, device=_lib.device())
    ws = _lib.workspace(_lib.ws_bytes(g, None, _lib.WS_RECONSTRUCT, _lib.I32))
    err = _lib.Err()
    _lib.call("hszg_recorrelate", ctypes.byref(g), _lib.ptr(p), _lib.ptr(meta) if meta is not None else None,
              _lib.ptr(out), _lib.I32, _lib.ptr(ws), ws.numel(), _lib.stream_handle(), ctypes.byref(err), err=err)
    values = out if isinstance(stream.values, t.Tensor) else out.cpu().numpy()
    return QuantizedField(values, stream.eps)


def _is_dev(x) -> bool:
    try:
        import torch

        return isinstance(x, torch.Tensor)
    except ImportError:  # pragma: no cover
        return False


def _clip_block_dims(block_dims, shape: GridShape) -> tuple:
    return tuple(min(b, n) for b, n in zip(block_dims, shape.dims))


def resolve_block_dims(kind: CompressorKind, shape: GridShape, block_dims) -> tuple:
    """Normalise user block dims to the stored per-axis form (compressors.py:245-270)."""
    if kind.is_nd:
        if shape.ndims < 2:
            raise ValueError(f"{kind.cli_name} requires 2D or 3D data")
        if block_dims is None:
            block_dims = DEFAULT_BLOCK_ND[shape.ndims]
        block_dims = tuple(int(b) for b in np.atleast_1d(block_dims))
        if len(block_dims) != shape.ndims:
            raise ValueError(f"{kind.cli_name} needs {shape.ndims} block extents, got {len(block_dims)}")
        return _clip_block_dims(block_dims, shape)
    if block_dims is None:
        size = DEFAULT_BLOCK_1D
    else:
        dims = tuple(int(b) for b in np.atleast_1d(block_dims))
        if len(dims) != 1:
            raise ValueError(f"{kind.cli_name} takes a single block size")
        size = dims[0]
    if size < 1:
        raise ValueError("block size must be >= 1")
    size = min(size, shape.total)
    return (size,) + (1,) * (shape.ndims - 1)


class CompressedStream:
    """Self-describing compressed container (compressors.py:273-310).

    Host fields (``payload`` bytes, ``chunk_offsets`` uint64, ``metadata``
    int32) and the device mirror (:meth:`device`) are each materialised on
    first use from whichever side the stream was created on.
    """

    def __init__(self, kind, shape, block_dims, eps, metadata=None, chunk_offsets=None, payload=None, *,
                 device: DeviceStream | None = None):
        self.kind = CompressorKind(kind)
        self.shape = shape if isinstance(shape, GridShape) else GridShape(tuple(shape))
        self.block_dims = tuple(int(b) for b in block_dims)
        self.eps = float(eps)
        self._metadata = metadata
        self._chunk_offsets = chunk_offsets
        self._payload = payload
        self._device = device
        if device is None and payload is None:
            raise ValueError("CompressedStream needs a host payload or a device mirror")

    # -- host views --------------------------------------------------------------
    @property
    def payload(self) -> bytes:
        if self._payload is None:
            d = self._device
            self._payload = d.payload[: d.payload_len].cpu().numpy().tobytes()
        return self._payload

    @payload.setter
    def payload(self, value):
        self._payload = value
        self._device = None
        self._pinned_payload = None

    @property
    def chunk_offsets(self) -> np.ndarray:
        if self._chunk_offsets is None:
            self._chunk_offsets = self._device.offsets.cpu().numpy().view(np.uint64).copy()
        return self._chunk_offsets

    @chunk_offsets.setter
    def chunk_offsets(self, value):
        self._chunk_offsets = value
        self._device = None

    @property
    def metadata(self):
        if self._metadata is None and self._device is not None and self._device.metadata is not None:
            self._metadata = self._device.metadata.cpu().numpy().copy()
        return self._metadata

    @metadata.setter
    def metadata(self, value):
        self._metadata = value
        self._device = None

    @property
    def payload_len(self) -> int:
        return self._device.payload_len if self._device is not None else len(self._payload)

    @property
    def n_chunks(self) -> int:
        if self._device is not None:
            return self._device.n_chunks
        return len(self._chunk_offsets)

    def pinned_payload(self):
        """The pinned torch buffer the payload views (streams from io.read_compressed), else None."""
        pin = getattr(self, "_pinned_payload", None)
        if pin is None or not isinstance(self._payload, memoryview) or pin.numel() != len(self._payload):
            return None
        return pin

    # -- device mirror -------------------------------------------------------------
    def device(self) -> DeviceStream:
        """The HBM-resident mirror (uploaded once, validated on first use)."""
        if self._device is None:
            self._device = DeviceStream.from_host(int(self.kind), self.shape.dims, self.block_dims, self.eps,
                                                  self._payload, self._chunk_offsets, self._metadata,
                                                  pinned_payload=self.pinned_payload())
        return self._device

    # -- geometry --------------------------------------------------------------------
    @cached_property
    def geometry(self) -> BlockGeometry:
        return effective_geometry(self.kind, self.shape, self.block_dims)

    @cached_property
    def spans(self) -> np.ndarray:
        return codec.spans_from_segments(segment_bounds(self.kind, self.shape, self.geometry))

    @cached_property
    def perm(self) -> np.ndarray:
        return stream_perm(self.kind, self.shape, self.geometry)

    @property
    def metadata_bytes(self) -> int:
        if not self.kind.is_block_mean:
            return 0
        return 4 * int(self.geometry.block_count)

    def byte_size(self) -> int:
        nd = self.shape.ndims
        header = 4 + 1 + 1 + 1 + 8 * nd + 4 * nd + 8 + 8
        index = 8 + 8 * self.n_chunks
        return header + 8 + self.metadata_bytes + index + self.payload_len

    def ratio(self) -> float:
        return 4.0 * self.shape.total / self.byte_size()


_ONE_PASS = os.environ.get("HSZG_COMPRESS", "") != "chain"      # "chain": the multi-kernel path (A/B, tests)
_TRIM_BYTES = 1 << 30                    # a worst-case payload buffer wasting more than this is trimmed


def _compress_one_pass(field_dev, kind: CompressorKind, shape: GridShape, eps: float, block_dims):
    """One kernel from the float32 field to the container (csrc/compress.cu, hszg_compress_fused), or None
    when the geometry has no one-pass front.  The payload is written into a worst-case buffer (its length
    is known only after the pass) that is trimmed to size when that wastes more than _TRIM_BYTES."""
    t = _lib.torch()
    if not eps > 0:
        raise ValueError(f"eps must be positive, got {eps}")
    g = _lib.make_geom(int(kind), shape.dims, block_dims, eps)
    wsb, cap = ctypes.c_uint64(0), ctypes.c_uint64(0)
    if not _lib.lib().hszg_compress_plan(ctypes.byref(g), ctypes.byref(wsb), ctypes.byref(cap)):
        return None
    flat = field_dev.reshape(-1)
    if int(flat.data_ptr()) % 16:
        return None
    dev = _lib.device()
    n_chunks = int(g.n_chunks)
    offs = t.empty(max(n_chunks, 1), dtype=t.int64, device=dev)[:n_chunks]
    meta = t.empty(max(int(g.n_blocks), 1), dtype=t.int32, device=dev) if kind.is_block_mean else None
    payload = t.empty(int(cap.value), dtype=t.uint8, device=dev)
    ws = _lib.workspace(int(wsb.value))
    total = ctypes.c_uint64(0)
    err = _lib.Err()
    _lib.call("hszg_compress_fused", ctypes.byref(g), _lib.ptr(flat), 1.0 / (2.0 * eps), _lib.ptr(payload),
              int(cap.value), _lib.ptr(offs), _lib.ptr(meta) if meta is not None else None, ctypes.byref(total),
              _lib.ptr(ws), ws.numel(), _lib.stream_handle(), ctypes.byref(err), err=err)
    plen = int(total.value)
    if payload.numel() - (plen + _lib.PAYLOAD_PAD) > _TRIM_BYTES:
        payload = payload[: plen + _lib.PAYLOAD_PAD].clone()
    if meta is not None:
        meta = meta[: int(g.n_blocks)]
    return DeviceStream(int(kind), shape.dims, block_dims, eps, payload, plen, offs, meta)


def compress_device(field_dev, kind: CompressorKind, eps: float, block_dims) -> DeviceStream:
    """Quantize + decorrelate + encode a CUDA float field into a DeviceStream (no host copies).  The
    decorrelation kernel also emits the chunk bit widths / sizes when every chunk is full
    (hszg_decorrelate_sized), so p is read once more only by the packer."""
    t = _lib.torch()
    kind = CompressorKind(kind)
    shape = GridShape(tuple(field_dev.shape))
    if field_dev.dtype == t.float32 and _ONE_PASS:
        ds = _compress_one_pass(field_dev, kind, shape, eps, block_dims)
        if ds is not None:
            return ds
    q = quantize_device(field_dev, eps)
    g = _lib.make_geom(int(kind), shape.dims, block_dims, eps)
    n_chunks = int(g.n_chunks)
    offs = t.empty(max(n_chunks, 1), dtype=t.int64, device=_lib.device())[:n_chunks]
    bws = t.empty(max(n_chunks, 1), dtype=t.uint8, device=_lib.device())
    p = t.empty(shape.total, dtype=t.int32, device=_lib.device())
    meta = t.empty(max(int(g.n_blocks), 1), dtype=t.int32, device=_lib.device()) if kind.is_block_mean else None
    fused = ctypes.c_int(0)
    err = _lib.Err()
    ws = _lib.workspace(256)
    _lib.call("hszg_decorrelate_sized", ctypes.byref(g), _lib.ptr(_as_device(q, t.int32).reshape(-1)), _lib.ptr(p),
              _lib.ptr(meta) if meta is not None else None, _lib.ptr(offs), _lib.ptr(bws), ctypes.byref(fused),
              _lib.ptr(ws), ws.numel(), _lib.stream_handle(), ctypes.byref(err), err=err)
    if meta is not None:
        meta = meta[: int(g.n_blocks)]
    del q
    total = ctypes.c_uint64(0)
    ws = _lib.workspace(_lib.ws_bytes(g, None, _lib.WS_ENCODE))
    if fused.value:
        _lib.call("hszg_encode_offsets", ctypes.byref(g), _lib.ptr(offs), ctypes.byref(total), _lib.ptr(ws),
                  ws.numel(), _lib.stream_handle(), ctypes.byref(err), err=err)
    else:
        _lib.call("hszg_encode_sizes", ctypes.byref(g), _lib.ptr(p), _lib.ptr(offs), _lib.ptr(bws),
                  ctypes.byref(total), _lib.ptr(ws), ws.numel(), _lib.stream_handle(), ctypes.byref(err), err=err)
    plen = int(total.value)
    payload = t.zeros(plen + _lib.PAYLOAD_PAD, dtype=t.uint8, device=_lib.device())
    _lib.call("hszg_encode_pack", ctypes.byref(g), _lib.ptr(p), _lib.ptr(offs), _lib.ptr(bws), _lib.ptr(payload),
              _lib.stream_handle(), ctypes.byref(err), err=err)
    del p, bws
    ds = DeviceStream(int(kind), shape.dims, block_dims, eps, payload, plen, offs, meta)
    return ds


@ranged("hsz/compress")
def compress(field, kind: CompressorKind, bound: ErrorBound, block_dims=None) -> CompressedStream:
    """Quantize, partition, decorrelate and encode a floating-point field (compressors.py:313-339)."""
    kind = CompressorKind(kind)
    d = _float_field(field)
    shape = GridShape(tuple(d.shape))
    _, _, bad = field_minmax(d.reshape(-1))
    if bad:
        raise ValueError("field contains NaN or Inf")
    eps = resolve_eps(d, bound)
    block_dims = resolve_block_dims(kind, shape, block_dims)
    ds = compress_device(d, kind, eps, block_dims)
    return CompressedStream(kind, shape, block_dims, eps, device=ds)
