"""Multi-stage partial decompression and slab streaming (reference hsz/stages.py).

Stages: 1 metadata, 2 decorrelated integers, 3 quantization indices, 4 floats.
``partial_decompress`` runs the fused sm_100a kernels on the stream's device
mirror (decode, prediction reversion, dequantization) and returns numpy
arrays by default, or CUDA tensors with ``out="torch"``.

Slabs are bands along axis 0 (one row/plane for HSZP_ND, one block-row for
HSZX_ND, one 1-D block for the flat kinds); chunks never cross slab
boundaries, so a slab is a self-contained sub-stream: the slab kernels run on
a view of the resident payload (same pointer, a slice of the chunk index and
of the metadata).  Prefix kinds carry the previous q row/plane/value between
slabs (stages.py:193-204), added on the device by ``hszg_add_plane``.
"""

from __future__ import annotations

import ctypes
import enum
import math
from dataclasses import dataclass

import numpy as np

from ._nvtx import ranged
from . import _lib
from .compressors import CompressedStream, CompressorKind, DecorrelatedStream
from .counters import decode_counters
from .device import DeviceStream
from .errors import UnsupportedStageError
from .quant import QuantizedField


class Stage(enum.IntEnum):
    META = 1
    DECORRELATED = 2
    QUANTIZED = 3
    FULL = 4

    @property
    def cli_name(self) -> str:
        return _STAGE_NAMES[self]

    @classmethod
    def from_name(cls, name: str) -> "Stage":
        for stage, label in _STAGE_NAMES.items():
            if label == name.strip().lower():
                return stage
        raise ValueError(f"unknown stage {name!r}")


_STAGE_NAMES = {
    Stage.META: "meta",
    Stage.DECORRELATED: "decorrelated",
    Stage.QUANTIZED: "quantized",
    Stage.FULL: "full",
}


def supported_stages(kind: CompressorKind) -> set:
    """stages.py:56-60."""
    stages = {Stage.DECORRELATED, Stage.QUANTIZED, Stage.FULL}
    if kind.is_block_mean:
        stages.add(Stage.META)
    return stages


def count_stage_work(c: CompressedStream, stage: Stage):
    """The reference's decode-work counter increments for one decompression (stages.py:73-87)."""
    if stage == Stage.META:
        decode_counters.bytes_read += c.metadata_bytes
        return
    decode_counters.chunks_decoded += c.n_chunks
    decode_counters.bytes_read += c.payload_len + c.metadata_bytes
    if stage >= Stage.QUANTIZED:
        decode_counters.recorrelated_elements += c.shape.total
    if stage == Stage.FULL:
        decode_counters.dequantized_elements += c.shape.total


def _check_stage(c: CompressedStream, stage: Stage):
    if stage not in supported_stages(c.kind):
        raise UnsupportedStageError(f"stage {stage.cli_name} is not supported by {c.kind.cli_name}")


@ranged("hsz/partial_decompress")
def partial_decompress(c: CompressedStream, stage: Stage, out: str = "numpy", dtype=None):
    """Decompress to ``stage`` (stages.py:63-88).

    Returns int32 metadata (1), a DecorrelatedStream (2), a QuantizedField
    (3) or a float64 grid (4; ``dtype=torch.float32`` for a float32 grid).
    """
    stage = Stage(stage)
    _check_stage(c, stage)
    t = _lib.torch()
    to_host = out == "numpy"
    if stage == Stage.META:
        count_stage_work(c, stage)
        if to_host:
            return np.array(c.metadata, copy=True)
        return c.device().metadata.clone()
    d = c.device()
    if stage == Stage.DECORRELATED:
        p = d.decode()
        count_stage_work(c, stage)
        meta = d.metadata
        if to_host:
            p = p.cpu().numpy()
            meta = None if meta is None else meta.cpu().numpy()
        return DecorrelatedStream(p, meta, c.geometry, c.shape, c.eps, c.kind, source=d)
    if stage == Stage.QUANTIZED:
        q = d.reconstruct(t.int32)
        count_stage_work(c, stage)
        return QuantizedField(q.cpu().numpy() if to_host else q, c.eps)
    f = d.reconstruct(dtype or t.float64)
    count_stage_work(c, stage)
    return f.cpu().numpy() if to_host else f


# ---------------------------------------------------------------------------
# Slab streaming


@dataclass
class SlabTracker:
    """Counts simultaneously live slab buffers (memory high-water proxy, stages.py:95-114)."""

    live: int = 0
    high_water: int = 0

    def alloc(self):
        self.live += 1
        self.high_water = max(self.high_water, self.live)

    def free(self):
        self.live -= 1

    def reset(self):
        self.live = 0
        self.high_water = 0


slab_tracker = SlabTracker()


def slab_bounds(c: CompressedStream) -> list:
    """Per-slab [start, end) along axis 0, flat positions for 1-D kinds (stages.py:117-128)."""
    if c.kind == CompressorKind.HSZP_ND:
        extent = 1
        n1 = c.shape.dims[0]
    elif c.kind == CompressorKind.HSZX_ND:
        extent = c.geometry.block_dims[0]
        n1 = c.shape.dims[0]
    else:
        extent = c.geometry.block_dims[0]
        n1 = c.shape.total
    return [(s, min(s + extent, n1)) for s in range(0, n1, extent)]


def _host_geom(c: CompressedStream):
    """The stream's geometry struct without uploading it (the device mirror's when it exists)."""
    if c._device is not None:
        return c._device.geom
    g = getattr(c, "_geom_cache", None)
    if g is None:
        g = _lib.make_geom(int(c.kind), c.shape.dims, c.block_dims, c.eps)
        c._geom_cache = g
    return g


def _slab_chunk_range(c: CompressedStream, lo: int, hi: int) -> tuple:
    """First/last chunk of slab rows [lo, hi): closed form (chunks restart per segment)."""
    g = _host_geom(c)
    if c.kind == CompressorKind.HSZP_ND:
        per = int(g.n_chunks) // c.shape.dims[0]       # every plane/row has the same chunk count
        return lo * per, hi * per
    if c.kind == CompressorKind.HSZX_ND:
        # a block-row of segments: chunks of all segments in rows [lo, hi)
        bd0 = c.geometry.block_dims[0]
        rows = -(-c.shape.dims[0] // bd0)
        full_row = _rowc(g, 0)
        b_lo = lo // bd0
        b_hi = -(-hi // bd0)
        first = b_lo * full_row
        last = first + sum(_rowc(g, int(b == rows - 1)) for b in range(b_lo, b_hi))
        return first, last
    S = c.geometry.block_dims[0]
    cps = -(-S // 32)
    b_lo = lo // S
    first = b_lo * cps
    last = first + -(-(hi - lo) // 32)
    return first, last


_ROWC_CACHE: dict = {}


def _rowc(g, edge: int) -> int:
    """Chunks in one block-row (all segments of one first-axis block index) of an HSZX_ND stream
    (memoised per geometry: slab iteration asks for it once per slab)."""
    key = (int(g.ndims), tuple(int(g.dims[k]) for k in range(g.ndims)),
           tuple(int(g.block_dims[k]) for k in range(g.ndims)), int(edge))
    v = _ROWC_CACHE.get(key)
    if v is None:
        v = _ROWC_CACHE[key] = _rowc_compute(g, edge)
    return v


def _rowc_compute(g, edge: int) -> int:
    nd = g.ndims
    dims = [g.dims[k] for k in range(nd)]
    bds = [g.block_dims[k] for k in range(nd)]
    s0 = dims[0] - (-(-dims[0] // bds[0]) - 1) * bds[0] if edge else bds[0]
    total = 0
    grids = [-(-dims[k] // bds[k]) for k in range(1, nd)]
    for idx in np.ndindex(*grids):
        size = s0
        for k, b in enumerate(idx, start=1):
            size *= bds[k] if b < grids[k - 1] - 1 else dims[k] - (grids[k - 1] - 1) * bds[k]
        total += -(-size // 32)
    return total


def _slab_layout(c: CompressedStream, lo: int, hi: int) -> tuple:
    """(first chunk, last chunk, metadata [lo, hi), dims, block dims) of slab rows [lo, hi)."""
    first, last = _slab_chunk_range(c, lo, hi)
    if c.kind.is_nd:
        dims = (hi - lo,) + tuple(c.shape.dims[1:])
        bd = tuple(min(b, n) for b, n in zip(c.block_dims, dims))
    else:
        dims = (hi - lo,)
        bd = (min(c.block_dims[0], hi - lo),)
    mlo = mhi = 0
    if c.kind.is_block_mean:
        if c.kind == CompressorKind.HSZX_ND:
            per_row = int(np.prod([-(-n // b) for n, b in zip(c.shape.dims[1:], c.block_dims[1:])]))
            b0 = lo // c.block_dims[0]
            mlo, mhi = b0 * per_row, (b0 + 1) * per_row
        else:
            S = c.block_dims[0]
            mlo, mhi = lo // S, lo // S + 1
    return first, last, mlo, mhi, dims, bd


def _slab_view(c: CompressedStream, lo: int, hi: int):
    """(DeviceStream over the slab's chunks, chunk count, payload bytes): same payload pointer,
    sliced chunk index and metadata, payload length cut at the slab's last byte."""
    d = c.device().validate()
    first, last, mlo, mhi, dims, bd = _slab_layout(c, lo, hi)
    offs = d.offsets[first:last]
    host = c.chunk_offsets            # host copy of the index (downloaded once): no per-slab sync
    end = int(host[last]) if last < d.n_chunks else d.payload_len
    meta = d.metadata[mlo:mhi] if c.kind.is_block_mean else None
    sub = DeviceStream.__new__(DeviceStream)
    DeviceStream.__init__(sub, int(c.kind), dims, bd, c.eps, d.payload, end, offs, meta)
    sub.desc.canonical = d.desc.canonical
    sub.desc.max_bitwidth = d.desc.max_bitwidth
    sub.validated = True
    return sub, last - first, end - (int(host[first]) if first < d.n_chunks else end)


def slab_iter(c: CompressedStream, stage: Stage, out: str = "numpy", from_host=None,
              budget: int | None = None):
    """Yield per-slab views in axis-0 order (stages.py:173-225); concatenation == whole stage.

    ``from_host=True`` streams the container from (pinned) host memory unit by unit instead of
    uploading it whole (streaming.HostSlabSource); ``None`` decides by size
    (streaming.should_stream).  Results are identical either way.
    """
    from . import streaming

    stage = Stage(stage)
    if stage not in supported_stages(c.kind) or stage == Stage.META:
        raise UnsupportedStageError(f"stage {stage.cli_name} is not slab-iterable for {c.kind.cli_name}")
    bounds = slab_bounds(c)
    src = None
    if streaming.should_stream(c, from_host):
        src = streaming.HostSlabSource(c, bounds, lambda lo, hi: _slab_layout(c, lo, hi),
                                       budget or streaming.DEFAULT_BUDGET)
    yield from _slab_iter_batched(c, stage, out, bounds, src)


SLAB_BATCH_BYTES = 64 << 20     # device bytes of int32 values decoded per launch group by slab_iter


def _slab_iter_batched(c: CompressedStream, stage: Stage, out: str, bounds: list, src=None):
    """slab_iter with consecutive slabs decoded together — up to SLAB_BATCH_BYTES of values per reconstruct
    launch and, when streaming from host memory, inside one fetch unit (HSZP_ND: one plane per slab would
    otherwise be one band-scan launch per plane) — and yielded as views of the batch: the same arrays,
    counters and slab-tracker events per slab as one-slab decoding (stages.py:173-225)."""
    t = _lib.torch()
    per_row = int(np.prod(c.shape.dims[1:])) if c.kind.is_nd else 1
    if src is None:
        host = c.chunk_offsets
        d = c.device().validate()
        nc, plen = d.n_chunks, d.payload_len

    def slab_bytes(k, lo, hi):
        if src is not None:                          # from the fetch units' slab table
            first, last, b0, b1 = src.slabs[k][:4]
            return last - first, b1 - b0
        first, last = _slab_chunk_range(c, lo, hi)
        a = int(host[first]) if first < nc else plen
        b = int(host[last]) if last < nc else plen
        return last - first, b - a

    carry = None
    cur_unit = -1
    k = 0
    while k < len(bounds):
        j = k + 1
        while (j < len(bounds) and (bounds[j][1] - bounds[k][0]) * per_row * 4 <= SLAB_BATCH_BYTES
               and (src is None or src.unit_of[j] == src.unit_of[k])):
            j += 1
        blo, bhi = bounds[k][0], bounds[j - 1][1]
        if src is None:
            sub, _, _ = _slab_view(c, blo, bhi)
        else:
            u = int(src.unit_of[k])
            if u != cur_unit and cur_unit >= 0:
                src.release(cur_unit)                # its slabs' kernels are queued: the slot may refill
            cur_unit = u
            sub = src.span(k, j)
        if stage == Stage.DECORRELATED:
            vals = sub.decode()
        elif c.kind == CompressorKind.HSZP_ND and carry is not None and sub.carry_ok():
            # the previous batch's last plane folded into this batch's z prefix (no separate add pass)
            vals = sub.reconstruct(t.int32, carry=carry)
            carry = vals.reshape(bhi - blo, -1)[-1].clone()
            if stage == Stage.FULL:
                from .quant import dequantize_device

                vals = dequantize_device(vals, c.eps)
        else:
            vals = sub.reconstruct(t.int32)
            if c.kind == CompressorKind.HSZP:
                vals = vals.reshape(-1)
                if carry is not None:
                    _lib.call("hszg_add_plane", _lib.ptr(vals), _lib.ptr(carry), 1, vals.numel(), _lib.stream_handle())
                carry = vals[-1:].clone()
            elif c.kind == CompressorKind.HSZP_ND:
                if carry is not None:
                    _lib.call("hszg_add_plane", _lib.ptr(vals), _lib.ptr(carry), per_row, vals.numel(),
                              _lib.stream_handle())
                carry = vals.reshape(bhi - blo, -1)[-1].clone()
            if stage == Stage.FULL:
                from .quant import dequantize_device

                vals = dequantize_device(vals, c.eps)
        flat = vals.reshape(-1)
        host_vals = flat.cpu().numpy() if out == "numpy" else None
        for i, (lo, hi) in enumerate(bounds[k:j], start=k):
            nch, nbytes = slab_bytes(i, lo, hi)
            decode_counters.chunks_decoded += nch
            decode_counters.bytes_read += nbytes
            a, b = (lo - blo) * per_row, (hi - blo) * per_row
            shape = ((hi - lo),) + tuple(c.shape.dims[1:]) if c.kind.is_nd else (hi - lo,)
            if stage != Stage.DECORRELATED:
                if c.kind.is_block_mean:
                    _, _, mlo, mhi, _, _ = _slab_layout(c, lo, hi)
                    decode_counters.bytes_read += 4 * (mhi - mlo)
                decode_counters.recorrelated_elements += b - a
                if stage == Stage.FULL:
                    decode_counters.dequantized_elements += b - a
            slab_tracker.alloc()
            if stage == Stage.DECORRELATED:                  # stage 2: stream order, flat (sub.decode())
                yield host_vals[a:b] if out == "numpy" else flat[a:b]
            else:
                yield host_vals[a:b].reshape(shape) if out == "numpy" else flat[a:b].reshape(shape)
        k = j


def sliding_window(c: CompressedStream, stage: Stage, out: str = "numpy", from_host=None):
    """Yield (index, prev, cur, nxt) slab triples holding at most 3 slabs (stages.py:228-258)."""
    it = slab_iter(c, stage, out, from_host=from_host)
    window: list = []
    try:
        window.append(next(it))
    except StopIteration:
        return
    nxt = next(it, None)
    if nxt is not None:
        window.append(nxt)
    idx = 0
    while True:
        prev = window[idx - 1] if idx > 0 else None
        cur = window[idx] if idx < len(window) else None
        if cur is None:
            return
        nxt = window[idx + 1] if idx + 1 < len(window) else None
        yield idx, prev, cur, nxt
        if nxt is None:
            return
        if idx > 0:
            window[idx - 1] = None
            slab_tracker.free()
        fetched = next(it, None)
        if fetched is not None:
            window.append(fetched)
        idx += 1
