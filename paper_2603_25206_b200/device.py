"""Device residency of a compressed stream and thin wrappers over the C ABI.

``DeviceStream`` is the HBM mirror of a ``CompressedStream``: the payload
(16-byte aligned, zero-padded), the chunk index and the block metadata,
uploaded once.  The first use validates every chunk on the GPU
(``hszg_validate``: the reference decoder's per-chunk checks,
_bitpack.pyx:110-140, plus a proof that the index is the encoder's exclusive
scan); later calls go straight to the fused kernels.  Everything here
returns CUDA tensors; conversion to numpy happens in the drop-in modules.
"""

from __future__ import annotations

import ctypes

import numpy as np

from . import _lib


def _t():
    return _lib.torch()


class DeviceStream:
    """A compressed stream resident in device memory."""

    def __init__(self, kind, dims, block_dims, eps, payload_dev, payload_len, offsets_dev, metadata_dev=None,
                 end_in_index: bool = False):
        t = _t()
        self.kind = int(kind)
        self.dims = tuple(int(d) for d in dims)
        self.block_dims = tuple(int(b) for b in block_dims)
        self.eps = float(eps)
        self.payload = payload_dev            # uint8, len >= payload_len + PAYLOAD_PAD, 16-B aligned
        self.payload_len = int(payload_len)
        self.offsets = offsets_dev            # int64 view of uint64 offsets
        self.metadata = metadata_dev          # int32 or None
        self.geom = _lib.make_geom(self.kind, self.dims, self.block_dims, self.eps)
        if self.offsets.numel() != self.geom.n_chunks:
            from .errors import CorruptStreamError

            raise CorruptStreamError("chunk index count disagrees with geometry")
        assert payload_dev.dtype == t.uint8 and payload_dev.is_cuda
        assert int(payload_dev.data_ptr()) % 16 == 0
        self.desc = _lib.StreamDesc()
        self.desc.payload = _lib.ptr(self.payload)
        # views of a longer resident index read their end from offsets[n_chunks] (no host sync)
        self.desc.payload_len = (1 << 63) if end_in_index else self.payload_len
        self.desc.offsets = _lib.ptr(self.offsets)
        self.desc.metadata = _lib.ptr(self.metadata) if self.metadata is not None else None
        self.desc.canonical = 0
        self.desc.max_bitwidth = 32
        self.validated = False

    # ---- construction -----------------------------------------------------------

    @classmethod
    def from_host(cls, kind, dims, block_dims, eps, payload: bytes, offsets, metadata=None, pinned_payload=None):
        t = _t()
        dev = _lib.device()
        n = len(payload)
        buf = t.zeros(n + _lib.PAYLOAD_PAD, dtype=t.uint8, device=dev)
        if n:
            if pinned_payload is not None:                   # in-place DMA from the pinned file buffer
                buf[:n].copy_(pinned_payload[:n], non_blocking=True)
            else:
                host = t.frombuffer(bytearray(payload), dtype=t.uint8)
                buf[:n].copy_(host)
        offs = np.ascontiguousarray(np.asarray(offsets, dtype=np.uint64)).view(np.int64)
        offs_dev = t.from_numpy(offs.copy()).to(dev)
        meta_dev = None
        if metadata is not None:
            meta_dev = t.from_numpy(np.ascontiguousarray(metadata, dtype=np.int32)).to(dev)
        return cls(kind, dims, block_dims, eps, buf, n, offs_dev, meta_dev)

    @property
    def n(self) -> int:
        return int(self.geom.n)

    @property
    def n_chunks(self) -> int:
        return int(self.geom.n_chunks)

    def nbytes(self) -> int:
        """Container bytes resident on the device (payload + index + metadata)."""
        meta = 0 if self.metadata is None else self.metadata.numel() * 4
        return self.payload_len + self.n_chunks * 8 + meta

    def plane_view(self, s: int, e: int) -> "DeviceStream":
        """Sub-stream of axis-0 planes [s, e) of a 2-D/3-D HSZP_ND or HSZX_ND stream (zero-copy).

        Chunks restart at every segment (compressors.py:105-119), so the planes form a contiguous chunk
        range: same payload pointer, a slice of the index and of the metadata, and the payload length cut
        at the range's last byte.  HSZX_ND ranges must be block-row aligned.
        """
        n0 = self.dims[0]
        if not (0 <= s < e <= n0):
            raise ValueError(f"plane range [{s}, {e}) outside [0, {n0})")
        nc = self.n_chunks
        if self.kind == 1:
            cpp = nc // n0
            first, last = s * cpp, e * cpp
            meta = None
        elif self.kind == 3:
            b0 = self.block_dims[0]
            if s % b0 or (e % b0 and e != n0):
                raise ValueError("HSZX_ND plane ranges must be block-row aligned")
            g = self.geom
            per_row_blocks = int(g.sgrid[1] * g.sgrid[2])
            if not hasattr(self, "_row_chunks"):
                self._row_chunks = _full_row_chunks(self)
            full_row_chunks = self._row_chunks
            first = (s // b0) * full_row_chunks
            last = (e // b0) * full_row_chunks if e < n0 else nc
            meta = self.metadata[(s // b0) * per_row_blocks:(-(-e // b0)) * per_row_blocks]
        else:
            raise ValueError("plane views need an nd kind")
        offs = self.offsets[first:last]
        in_index = last < nc
        dims = (e - s,) + self.dims[1:]
        bd = tuple(min(b, n) for b, n in zip(self.block_dims, dims))
        sub = DeviceStream(self.kind, dims, bd, self.eps, self.payload, self.payload_len, offs, meta,
                           end_in_index=in_index or self.desc.payload_len == (1 << 63))
        sub.desc.canonical = self.desc.canonical
        sub.desc.max_bitwidth = self.desc.max_bitwidth
        sub.validated = self.validated
        return sub

    def mean_absmax(self) -> int:
        """max |M_b| over the block means (cached; 0 without metadata): with the max bit width it bounds
        |q| = |p + M_b| for the int32 stencil kernels (fused, table emitter)."""
        if getattr(self, "_mean_absmax", None) is None:
            m = self.metadata
            self._mean_absmax = 0 if m is None or m.numel() == 0 else int(m.to(_lib.torch().int64).abs().max())
        return self._mean_absmax

    # ---- validation -----------------------------------------------------------------

    def validate(self):
        if self.validated:
            return self
        err = _lib.Err()
        ws = _lib.workspace(_lib.ws_bytes(self.geom, None, _lib.WS_VALIDATE))
        _lib.call("hszg_validate", ctypes.byref(self.geom), ctypes.byref(self.desc), _lib.ptr(ws), ws.numel(),
                  _lib.stream_handle(), ctypes.byref(err), err=err)
        self.validated = True
        return self

    # ---- stages ------------------------------------------------------------------

    def decode(self, out=None):
        """Stage 2: int32 residuals in stream order."""
        t = _t()
        self.validate()
        if out is None:
            out = t.empty(self.n, dtype=t.int32, device=_lib.device())
        err = _lib.Err()
        _lib.call("hszg_decode", ctypes.byref(self.geom), ctypes.byref(self.desc), _lib.ptr(out),
                  _lib.stream_handle(), ctypes.byref(err), err=err)
        return out

    def reconstruct(self, dtype=None, out=None, carry=None):
        """Stage 3 (int32 q, row-major grid) or stage 4 (float32/float64 q*2eps).  carry: q of the plane before
        this sub-stream's first (3-D HSZP_ND slabs, `carry_ok`), folded into the z prefix."""
        t = _t()
        self.validate()
        dtype = dtype or t.int32
        code = {t.int32: _lib.I32, t.float32: _lib.F32, t.float64: _lib.F64}[dtype]
        if out is None:
            out = t.empty(self.dims, dtype=dtype, device=_lib.device())
        ws = _lib.workspace(_lib.ws_bytes(self.geom, self.desc, _lib.WS_RECONSTRUCT, code))
        err = _lib.Err()
        if carry is None:
            _lib.call("hszg_reconstruct", ctypes.byref(self.geom), ctypes.byref(self.desc), _lib.ptr(out), code,
                      _lib.ptr(ws), ws.numel(), _lib.stream_handle(), ctypes.byref(err), err=err)
        else:
            _lib.call("hszg_reconstruct_carry", ctypes.byref(self.geom), ctypes.byref(self.desc), _lib.ptr(out), code,
                      _lib.ptr(carry), _lib.ptr(ws), ws.numel(), _lib.stream_handle(), ctypes.byref(err), err=err)
        return out

    def carry_ok(self) -> bool:
        """reconstruct(carry=...) applies: a canonical 3-D HSZP_ND stream whose rows are whole chunks."""
        self.validate()
        return (self.kind == 1 and len(self.dims) == 3 and bool(self.desc.canonical) and self.dims[2] % 32 == 0
                and self.dims[2] <= 4096 and self.dims[0] <= 65535)

    # ---- reductions --------------------------------------------------------------

    def quantized_sums(self, out=None):
        """Exact sums of stage-3 q without writing q (hszg_quantized_sums), or None when this stream
        has no fused path (the caller reconstructs and reduces)."""
        self.validate()
        n = _lib.ws_bytes(self.geom, self.desc, _lib.WS_QSUMS)
        if n == 0:
            return None
        out = _lib.sums_tensor() if out is None else out
        ws = _lib.workspace(n)
        err = _lib.Err()
        _lib.call("hszg_quantized_sums", ctypes.byref(self.geom), ctypes.byref(self.desc), _lib.ptr(out),
                  _lib.ptr(ws), ws.numel(), _lib.stream_handle(), ctypes.byref(err), err=err)
        return out

    def reduce(self, mode: int, out=None):
        """Fused reduction from the compressed bytes (see hszg_reduce_stream); device Sums buffer."""
        self.validate()
        out = _lib.sums_tensor() if out is None else out
        ws = _lib.workspace(_lib.ws_bytes(self.geom, self.desc, _lib.WS_REDUCE))
        err = _lib.Err()
        _lib.call("hszg_reduce_stream", ctypes.byref(self.geom), ctypes.byref(self.desc), int(mode), _lib.ptr(out),
                  _lib.ptr(ws), ws.numel(), _lib.stream_handle(), ctypes.byref(err), err=err)
        return out


def _full_row_chunks(ds: DeviceStream) -> int:
    """Chunks in one full-thickness block-row of an HSZX_ND stream (closed form, host side)."""
    if ds.dims[0] <= ds.block_dims[0]:
        return ds.n_chunks
    # first chunk of block-row 1 = chunks of block-row 0; found by bisection on the chunk starts
    row_elems = ds.block_dims[0] * int(np.prod(ds.dims[1:]))
    lo, hi = 0, ds.n_chunks
    while lo < hi:
        mid = (lo + hi) // 2
        s, _, _ = _lib.locate_chunks(ds.geom, mid, 1)
        if s[0] < row_elems:
            lo = mid + 1
        else:
            hi = mid
    return lo


# ---------------------------------------------------------------------------
# array-level helpers (int32 CUDA tensors)

REDUCE_WS = 148 * 16 * 64 + 4096


def reduce_i32(x, out=None):
    out = _lib.sums_tensor() if out is None else out
    x = x.reshape(-1).contiguous()
    ws = _lib.workspace(REDUCE_WS)
    _lib.call("hszg_reduce_i32", _lib.ptr(x), x.numel(), _lib.ptr(out), _lib.ptr(ws), ws.numel(), _lib.stream_handle())
    return out


def reduce_dot(a, b, out=None):
    out = _lib.sums_tensor() if out is None else out
    a = a.reshape(-1).contiguous()
    b = b.reshape(-1).contiguous()
    ws = _lib.workspace(REDUCE_WS)
    _lib.call("hszg_reduce_dot", _lib.ptr(a), _lib.ptr(b), a.numel(), _lib.ptr(out), _lib.ptr(ws), ws.numel(),
              _lib.stream_handle())
    return out


def reduce_f64(q, scale, mean_dev=None, out=None):
    out = _lib.sums_tensor() if out is None else out
    q = q.reshape(-1).contiguous()
    ws = _lib.workspace(REDUCE_WS)
    _lib.call("hszg_reduce_f64", _lib.ptr(q), q.numel(), float(scale), _lib.ptr(mean_dev) if mean_dev is not None else None,
              _lib.ptr(out), _lib.ptr(ws), ws.numel(), _lib.stream_handle())
    return out


def reduce_array(geom, p, metadata, mode, out=None):
    out = _lib.sums_tensor() if out is None else out
    ws = _lib.workspace(REDUCE_WS)
    _lib.call("hszg_reduce_array", ctypes.byref(geom), _lib.ptr(p), _lib.ptr(metadata) if metadata is not None else None,
              int(mode), _lib.ptr(out), _lib.ptr(ws), ws.numel(), _lib.stream_handle())
    return out


def _nout(op, nd, ncomp):
    if op == _lib.OP_DERIV:
        return nd
    if op == _lib.OP_GRAD_LAP:
        return nd + 1
    if op == _lib.OP_CURL:
        return 1 if ncomp == 2 else 3
    return 1


def _stencil_arrays(q_list, eps_list, outs):
    dims = tuple(q_list[0].shape)
    nd = len(dims)
    ncomp = len(q_list)
    dims_arr = (ctypes.c_int64 * 3)(*(list(dims) + [1] * (3 - nd)))
    qptr = (ctypes.c_void_p * 3)(*([_lib.ptr(q) for q in q_list] + [None] * (3 - ncomp)))
    eps_arr = (ctypes.c_double * 3)(*(list(map(float, eps_list)) + [0.0] * (3 - ncomp)))
    optr = (ctypes.c_void_p * 4)(*([_lib.ptr(o) for o in outs] + [None] * (4 - len(outs))))
    return dims_arr, qptr, eps_arr, optr


def stencil(op, q_list, eps_list, float_domain=False, dtype=None, outs=None):
    """Run one K-STEN op over int32 (or float64, float_domain=2) grids; returns the output tensors."""
    t = _t()
    dtype = dtype or t.float64
    code = _lib.F32 if dtype == t.float32 else _lib.F64
    dims = tuple(q_list[0].shape)
    nd = len(dims)
    nout = _nout(op, nd, len(q_list))
    if outs is None:
        outs = [t.empty(dims, dtype=dtype, device=_lib.device()) for _ in range(nout)]
    qs = [q.contiguous() for q in q_list]
    dims_arr, qptr, eps_arr, optr = _stencil_arrays(qs, eps_list, outs)
    _lib.call("hszg_stencil", int(op), nd, ctypes.cast(dims_arr, ctypes.c_void_p), len(qs),
              ctypes.cast(qptr, ctypes.c_void_p), ctypes.cast(eps_arr, ctypes.c_void_p), int(float_domain),
              code, ctypes.cast(optr, ctypes.c_void_p), _lib.stream_handle())
    return outs


def stencil_window(op, q_list, eps_list, outs, zlo, zhi, gz0, gN0, float_domain=False):
    """3-D stencil over box planes [zlo, zhi) of q (plane 0 at global z = gz0 of gN0 planes) into outs."""
    t = _t()
    code = _lib.F32 if outs[0].dtype == t.float32 else _lib.F64
    dims_arr, qptr, eps_arr, optr = _stencil_arrays(q_list, eps_list, outs)
    _lib.call("hszg_stencil_window", int(op), ctypes.cast(dims_arr, ctypes.c_void_p), len(q_list),
              ctypes.cast(qptr, ctypes.c_void_p), ctypes.cast(eps_arr, ctypes.c_void_p), int(float_domain), code,
              ctypes.cast(optr, ctypes.c_void_p), int(zlo), int(zhi), int(gz0), int(gN0), _lib.stream_handle())
    return outs


def sums_combine(parts_buf, n, out=None):
    """Combine n consecutive HszgSums records (uint8 CUDA buffer) into one."""
    out = _lib.sums_tensor() if out is None else out
    _lib.call("hszg_sums_combine", _lib.ptr(parts_buf), int(n), _lib.ptr(out), _lib.stream_handle())
    return out


REGION_WORDS = 9   # 8-byte words per region in region_buffer (+1 trailing word: the crossing count)


def region_buffer(nr):
    """One int64 device buffer holding every per-region output, so the host reads it in one copy:
    words [k*nr, (k+1)*nr) for k = 0 s1, 1 s2 low, 2 s2 high, 3 size, 4 mean, 5 var, 6 vmin, 7 vmax
    (float64 bits), 8 qmin|qmax (2*nr int32), then the count."""
    return _t().empty(REGION_WORDS * nr + 1, dtype=_t().int64, device=_lib.device())


def region_views(buf, nr):
    t = _t()
    w = [buf[k * nr:(k + 1) * nr] for k in range(REGION_WORDS)]
    mm = w[8].view(t.int32)
    return dict(s1=w[0], s2lo=w[1], s2hi=w[2], size=w[3], mean=w[4].view(t.float64), var=w[5].view(t.float64),
                vmin=w[6].view(t.float64), vmax=w[7].view(t.float64), qmin=mm[:nr], qmax=mm[nr:],
                count=buf[REGION_WORDS * nr:])


def region_reduce(q, region, buf=None):
    """Per-region exact (S1, S2, qmin, qmax, size) over an int32 grid (N2-N4), into region_buffer."""
    dims = tuple(q.shape)
    nd = len(dims)
    reg = tuple(min(int(r), int(n)) for r, n in zip(region, dims))
    grid = tuple(-(-n // r) for n, r in zip(dims, reg))
    nr = int(np.prod(grid))
    buf = region_buffer(nr) if buf is None else buf
    v = region_views(buf, nr)
    dims_arr = (ctypes.c_int64 * 3)(*(list(dims) + [1] * (3 - nd)))
    reg_arr = (ctypes.c_int64 * 3)(*(list(reg) + [1] * (3 - nd)))
    qc = q.contiguous()
    _lib.call("hszg_region_reduce", _lib.ptr(qc), nd, ctypes.cast(dims_arr, ctypes.c_void_p),
              ctypes.cast(reg_arr, ctypes.c_void_p), _lib.ptr(v["s1"]), _lib.ptr(v["s2lo"]), _lib.ptr(v["s2hi"]),
              _lib.ptr(v["qmin"]), _lib.ptr(v["qmax"]), _lib.ptr(v["size"]), _lib.stream_handle())
    return grid, buf, v
