"""ORACLE — test infrastructure only (see oracle/__init__.py).

numpy + plain-C restatement of the reference HSZ pipeline.  Every function
cites the reference location it restates (paths relative to
/root/reference/pkg/src/hsz/).  Integer work is exact (int64 with Python-int
fallbacks, as the reference does); floating-point finalisations use the
reference's own expression order so scalars come out bit-identical.
"""

from __future__ import annotations

import ctypes
import math
import os
import struct
import subprocess
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))

CHUNK_CAP = 32                      # codec.py:20
QMAX = 2**31 - 2                    # quant.py:19
PMAX = 2**31 - 1                    # compressors.py:22
DEFAULT_BLOCK_1D = 32               # compressors.py:25
DEFAULT_BLOCK_ND = {2: (8, 8), 3: (8, 8, 8)}   # compressors.py:26
INT64_HEADROOM = 2**62              # analytics/stats.py:20

HSZP, HSZP_ND, HSZX, HSZX_ND = 0, 1, 2, 3       # compressors.py:29-33
KIND_NAMES = {HSZP: "hszp", HSZP_ND: "hszp-nd", HSZX: "hszx", HSZX_ND: "hszx-nd"}
META, DECORRELATED, QUANTIZED, FULL = 1, 2, 3, 4  # stages.py:30-34


def is_nd(kind):
    return kind in (HSZP_ND, HSZX_ND)


def is_block_mean(kind):
    return kind in (HSZX, HSZX_ND)


class OracleError(Exception):
    """Raised with the reference's exception class name and message."""

    def __init__(self, cls, msg):
        super().__init__(f"{cls}: {msg}")
        self.cls = cls
        self.msg = msg


# ---------------------------------------------------------------------------
# C codec (oracle/hsz_codec.c), built on demand


_LIB = None


def _lib():
    global _LIB
    if _LIB is not None:
        return _LIB
    path = os.path.join(HERE, "_build", "libhszoracle.so")
    src = os.path.join(HERE, "hsz_codec.c")
    if not os.path.exists(path) or os.path.getmtime(path) < os.path.getmtime(src):
        subprocess.run(["make", "-s", "-C", HERE], check=True)
    lib = ctypes.CDLL(path)
    i64p = ctypes.POINTER(ctypes.c_int64)
    lib.hszo_encode_sizes.restype = ctypes.c_int64
    lib.hszo_encode_sizes.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                                      ctypes.c_int64, ctypes.c_void_p, ctypes.c_void_p, i64p]
    lib.hszo_encode_pack.restype = None
    lib.hszo_encode_pack.argtypes = [ctypes.c_void_p] * 3 + [ctypes.c_int64] + [ctypes.c_void_p] * 3
    lib.hszo_decode.restype = ctypes.c_int
    lib.hszo_decode.argtypes = [ctypes.c_void_p, ctypes.c_uint64, ctypes.c_void_p, ctypes.c_void_p,
                                ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p, i64p, i64p]
    lib.hszo_num_threads.restype = ctypes.c_int
    lib.hszo_set_threads.argtypes = [ctypes.c_int]
    _LIB = lib
    return lib


def set_threads(n):
    _lib().hszo_set_threads(int(n))


def num_threads():
    return _lib().hszo_num_threads()


def _ptr(a):
    return a.ctypes.data_as(ctypes.c_void_p)


def encode_stream(values, spans):
    """_kernels.encode_stream (_bitpack.pyx:14-87): returns (payload bytes, uint64 offsets)."""
    vals = np.ascontiguousarray(values, dtype=np.int32)
    starts = np.ascontiguousarray(spans[:, 0], dtype=np.int64)
    ends = np.ascontiguousarray(spans[:, 1], dtype=np.int64)
    n = len(starts)
    bws = np.zeros(n, dtype=np.uint8)
    offsets = np.zeros(n, dtype=np.uint64)
    bad = ctypes.c_int64(-1)
    lib = _lib()
    total = lib.hszo_encode_sizes(_ptr(vals), _ptr(starts), _ptr(ends), n, _ptr(bws),
                                  _ptr(offsets), ctypes.byref(bad))
    if total < 0:
        raise OracleError("ValueError", "value -2**31 has no sign-magnitude representation")
    out = np.zeros(int(total), dtype=np.uint8)
    lib.hszo_encode_pack(_ptr(vals), _ptr(starts), _ptr(ends), n, _ptr(bws), _ptr(offsets), _ptr(out))
    return out.tobytes(), offsets


_DECODE_MSGS = {
    1: "chunk offset past end of payload",      # _bitpack.pyx:112
    2: None,                                    # _bitpack.pyx:115 (formatted)
    3: "truncated chunk payload",               # _bitpack.pyx:123
    4: "chunk magnitude exceeds int32 range",   # _bitpack.pyx:136
    5: "negative zero in chunk",                # _bitpack.pyx:140
}


def decode_stream(payload, spans, offsets):
    """_kernels.decode_stream (_bitpack.pyx:90-144): int32 values in stream order."""
    buf = np.frombuffer(bytes(payload), dtype=np.uint8) if not isinstance(payload, np.ndarray) else payload
    buf = np.ascontiguousarray(buf, dtype=np.uint8)
    starts = np.ascontiguousarray(spans[:, 0], dtype=np.int64)
    ends = np.ascontiguousarray(spans[:, 1], dtype=np.int64)
    offs = np.ascontiguousarray(offsets, dtype=np.uint64)
    n = int(ends[-1]) if len(ends) else 0
    out = np.zeros(n, dtype=np.int32)
    bc, be = ctypes.c_int64(-1), ctypes.c_int64(-1)
    kind = _lib().hszo_decode(_ptr(buf) if buf.size else None, buf.size, _ptr(starts), _ptr(ends),
                              _ptr(offs), len(starts), _ptr(out), ctypes.byref(bc), ctypes.byref(be))
    if kind:
        if kind == 2:
            off = int(offs[bc.value])
            raise OracleError("CorruptStreamError", f"chunk bitwidth {int(buf[off])} exceeds 32")
        raise OracleError("CorruptStreamError", _DECODE_MSGS[kind])
    return out


def chunk_byte_size(count, bitwidth):
    """_fallback.py:52-55."""
    if bitwidth == 0:
        return 1
    return 1 + (count + 7) // 8 + (count * bitwidth + 7) // 8


# ---------------------------------------------------------------------------
# Geometry (grid.py, compressors.py)


def block_grid(dims, block_dims):
    """grid.py:110."""
    return tuple(-(-n // b) for n, b in zip(dims, block_dims))


def block_sizes(dims, block_dims):
    """BlockGeometry.block_sizes (grid.py:72-81)."""
    g = block_grid(dims, block_dims)
    per_axis = [np.minimum((np.arange(gg) + 1) * bd, n) - np.arange(gg) * bd
                for gg, bd, n in zip(g, block_dims, dims)]
    sizes = per_axis[0]
    for ax in per_axis[1:]:
        sizes = np.multiply.outer(sizes, ax)
    return np.asarray(sizes).ravel().astype(np.int64)


def block_contiguous_perm(dims, block_dims):
    """canonical_order(..., 'block-contiguous') (grid.py:114-128): stream pos -> flat index."""
    total = int(np.prod(dims))
    flat = np.arange(total, dtype=np.int64).reshape(dims)
    parts = []
    for b in np.ndindex(*block_grid(dims, block_dims)):
        sl = tuple(slice(i * bd, min((i + 1) * bd, n)) for i, bd, n in zip(b, block_dims, dims))
        parts.append(flat[sl].ravel())
    return np.concatenate(parts)


def clip_block_dims(block_dims, dims):
    """compressors.py:241-242."""
    return tuple(min(b, n) for b, n in zip(block_dims, dims))


def resolve_block_dims(kind, dims, block_dims=None):
    """compressors.py:245-270."""
    if is_nd(kind):
        if len(dims) < 2:
            raise OracleError("ValueError", f"{KIND_NAMES[kind]} requires 2D or 3D data")
        if block_dims is None:
            block_dims = DEFAULT_BLOCK_ND[len(dims)]
        block_dims = tuple(int(b) for b in np.atleast_1d(block_dims))
        if len(block_dims) != len(dims):
            raise OracleError("ValueError", "block extents mismatch")
        return clip_block_dims(block_dims, dims)
    if block_dims is None:
        size = DEFAULT_BLOCK_1D
    else:
        bd = tuple(int(b) for b in np.atleast_1d(block_dims))
        if len(bd) != 1:
            raise OracleError("ValueError", "single block size")
        size = bd[0]
    if size < 1:
        raise OracleError("ValueError", "block size must be >= 1")
    size = min(size, int(np.prod(dims)))
    return (size,) + (1,) * (len(dims) - 1)


def effective_geometry(kind, dims, block_dims):
    """compressors.py:87-93 -> (geometry dims, geometry block dims)."""
    if is_nd(kind):
        return tuple(dims), tuple(block_dims)
    return (int(np.prod(dims)),), (int(block_dims[0]),)


def segment_bounds(kind, dims, block_dims):
    """compressors.py:105-119."""
    if kind == HSZP_ND:
        slab = int(np.prod(dims[1:], dtype=np.int64))
        return [(i * slab, (i + 1) * slab) for i in range(dims[0])]
    gd, gb = effective_geometry(kind, dims, block_dims)
    sizes = block_sizes(gd, gb)
    ends = np.cumsum(sizes)
    starts = ends - sizes
    return list(zip(starts.tolist(), ends.tolist()))


def spans_from_segments(segments):
    """codec.py:96-106."""
    spans = []
    for s, e in segments:
        for c in range(s, e, CHUNK_CAP):
            spans.append((c, min(c + CHUNK_CAP, e)))
    return np.asarray(spans, dtype=np.int64).reshape(-1, 2)


def stream_spans(kind, dims, block_dims):
    return spans_from_segments(segment_bounds(kind, dims, block_dims))


def stream_perm(kind, dims, block_dims):
    """compressors.py:96-102 (identity except HSZX_ND)."""
    if kind == HSZX_ND:
        return block_contiguous_perm(dims, block_dims)
    return np.arange(int(np.prod(dims)), dtype=np.int64)


# ---------------------------------------------------------------------------
# Quantization (quant.py)


def resolve_eps(field, mode, requested):
    """quant.py:56-66."""
    if mode == "abs":
        return float(requested)
    lo = float(np.min(field))
    hi = float(np.max(field))
    if hi == lo:
        raise OracleError("ZeroValueRangeError",
                          "constant field has zero value range; use an absolute error bound")
    return float(requested) * (hi - lo)


def quantize(values, eps):
    """quant.py:69-82 (reciprocal form, no FMA: numpy evaluates mul then add)."""
    recip = 1.0 / (2.0 * eps)
    scaled = np.asarray(values, dtype=np.float64) * recip + 0.5
    q = np.floor(scaled)
    if np.any(np.abs(q) > QMAX):
        raise OracleError("EpsTooSmallError", f"quantization index exceeds {QMAX}; increase the error bound")
    return q.astype(np.int32)


def dequantize(q, eps):
    """quant.py:85-87 / stages.py:88."""
    return np.asarray(q, dtype=np.float64) * (2.0 * eps)


# ---------------------------------------------------------------------------
# Decorrelation (compressors.py)


def block_means(sums, sizes):
    """_block_means (compressors.py:134-138): truncation toward zero."""
    means = sums // sizes
    means[(sums < 0) & (sums % sizes != 0)] += 1
    return means


def check_residuals(p):
    """compressors.py:141-146."""
    if p.size and int(np.abs(p).max()) > PMAX:
        raise OracleError("EpsTooSmallError",
                          "decorrelated residual overflows 32-bit range; increase the error bound")
    return p.astype(np.int32)


def decorrelate(q, kind, block_dims):
    """decorrelate (compressors.py:229-238) -> (p stream int32, metadata int32 or None)."""
    dims = q.shape
    if kind == HSZP:                                   # compressors.py:149-157
        flat = q.ravel().astype(np.int64)
        return check_residuals(np.diff(flat, prepend=np.int64(0))), None
    if kind == HSZP_ND:                                # compressors.py:160-176
        r = q.astype(np.int64)
        for ax in range(q.ndim):
            r = np.diff(r, axis=ax, prepend=np.int64(0))
        return check_residuals(r.ravel()), None
    gd, gb = effective_geometry(kind, dims, block_dims)  # compressors.py:179-198
    perm = stream_perm(kind, gd if kind == HSZX else dims, gb)
    stream = q.ravel().astype(np.int64)[perm]
    sizes = block_sizes(gd, gb)
    starts = np.concatenate(([0], np.cumsum(sizes)[:-1]))
    sums = np.add.reduceat(stream, starts)
    means = block_means(sums, sizes)
    p = stream - np.repeat(means, sizes)
    return check_residuals(p), means.astype(np.int32)


def recorrelate(p, metadata, kind, dims, block_dims):
    """compressors.py:201-226 -> int32 grid (row-major)."""
    if kind == HSZP:
        q = np.cumsum(p.astype(np.int64)).reshape(dims)
    elif kind == HSZP_ND:
        q = p.astype(np.int64).reshape(dims)
        for ax in range(len(dims)):
            q = np.cumsum(q, axis=ax)
    else:
        gd, gb = effective_geometry(kind, dims, block_dims)
        sizes = block_sizes(gd, gb)
        q_stream = p.astype(np.int64) + np.repeat(metadata.astype(np.int64), sizes)
        perm = stream_perm(kind, dims, block_dims)
        flat = np.empty(int(np.prod(dims)), dtype=np.int64)
        flat[perm] = q_stream
        q = flat.reshape(dims)
    return q.astype(np.int32)


def as_grid(p, kind, dims, block_dims):
    """DecorrelatedStream.as_grid (compressors.py:68-73)."""
    perm = stream_perm(kind, dims, block_dims)
    out = np.empty(int(np.prod(dims)), dtype=np.int32)
    out[perm] = p
    return out.reshape(dims)


def metadata_grid(metadata, kind, dims, block_dims):
    """DecorrelatedStream.metadata_grid (compressors.py:75-84)."""
    gd, gb = effective_geometry(kind, dims, block_dims)
    per_point = np.repeat(metadata.astype(np.int64), block_sizes(gd, gb))
    perm = stream_perm(kind, dims, block_dims)
    out = np.empty(int(np.prod(dims)), dtype=np.int64)
    out[perm] = per_point
    return out.reshape(dims)


# ---------------------------------------------------------------------------
# Container (compressors.CompressedStream + io.py)


@dataclass
class Stream:
    kind: int
    dims: tuple
    block_dims: tuple
    eps: float
    metadata: np.ndarray | None
    offsets: np.ndarray
    payload: bytes

    @property
    def n(self):
        return int(np.prod(self.dims))

    @property
    def spans(self):
        return stream_spans(self.kind, self.dims, self.block_dims)


def compress(field, kind, mode, requested, block_dims=None):
    """compress (compressors.py:313-339)."""
    field = np.asarray(field)
    if not np.all(np.isfinite(field)):
        raise OracleError("ValueError", "field contains NaN or Inf")
    eps = resolve_eps(field, mode, requested)
    q = quantize(field, eps)
    bd = resolve_block_dims(kind, field.shape, block_dims)
    p, meta = decorrelate(q, kind, bd)
    payload, offsets = encode_stream(p, stream_spans(kind, field.shape, bd))
    return Stream(kind, tuple(field.shape), bd, eps, meta, offsets, payload)


def stream_to_bytes(c: Stream) -> bytes:
    """io.py:44-61 (HSZ1 container)."""
    nd = len(c.dims)
    out = bytearray(b"HSZ1")
    out += struct.pack("<BBB", 1, int(c.kind), nd)
    out += struct.pack(f"<{nd}Q", *c.dims)
    out += struct.pack(f"<{nd}I", *c.block_dims)
    out += struct.pack("<dQ", c.eps, c.n)
    meta = b"" if c.metadata is None else np.ascontiguousarray(c.metadata, dtype="<i4").tobytes()
    out += struct.pack("<Q", len(meta)) + meta
    index = np.ascontiguousarray(c.offsets, dtype="<u8").tobytes()
    out += struct.pack("<Q", len(index)) + index
    out += c.payload
    return bytes(out)


def stream_from_bytes(buf: bytes) -> Stream:
    """io.py:85-129 (validation subset used by the tests)."""
    pos = 0

    def take(n):
        nonlocal pos
        if pos + n > len(buf):
            raise OracleError("CorruptStreamError", "truncated container")
        out = buf[pos:pos + n]
        pos += n
        return out

    if take(4) != b"HSZ1":
        raise OracleError("CorruptStreamError", "bad magic; not an HSZ container")
    version, kind, nd = struct.unpack("<BBB", take(3))
    if version != 1:
        raise OracleError("CorruptStreamError", f"unsupported container version {version}")
    dims = struct.unpack(f"<{nd}Q", take(8 * nd))
    bd = struct.unpack(f"<{nd}I", take(4 * nd))
    eps, count = struct.unpack("<dQ", take(16))
    (ml,) = struct.unpack("<Q", take(8))
    meta = None if ml == 0 else np.frombuffer(take(ml), dtype="<i4").astype(np.int32)
    (il,) = struct.unpack("<Q", take(8))
    offs = np.frombuffer(take(il), dtype="<u8").astype(np.uint64)
    return Stream(kind, tuple(int(d) for d in dims), tuple(int(b) for b in bd), eps, meta, offs,
                  bytes(buf[pos:]))


# ---------------------------------------------------------------------------
# Stages (stages.py:63-88)


def stage2(c: Stream):
    return decode_stream(c.payload, c.spans, c.offsets)


def stage3(c: Stream, p=None):
    if p is None:
        p = stage2(c)
    return recorrelate(p, c.metadata, c.kind, c.dims, c.block_dims)


def stage4(c: Stream, q=None):
    if q is None:
        q = stage3(c)
    return q.astype(np.float64) * (2.0 * c.eps)


# ---------------------------------------------------------------------------
# Exact statistics (analytics/stats.py)


def exact_sum(values):
    """_exact_sum (stats.py:30-39)."""
    v = np.ascontiguousarray(values, dtype=np.int64).ravel()
    if v.size == 0:
        return 0
    bound = int(np.abs(v).max())
    if bound == 0:
        return 0
    step = max(1, INT64_HEADROOM // bound)
    return sum(int(v[i:i + step].sum()) for i in range(0, v.size, step))


def exact_dot(a, b):
    """_exact_dot (stats.py:42-55)."""
    a = np.ascontiguousarray(a, dtype=np.int64).ravel()
    b = np.ascontiguousarray(b, dtype=np.int64).ravel()
    if a.size == 0:
        return 0
    bound = int(np.abs(a).max()) * int(np.abs(b).max())
    if bound == 0:
        return 0
    step = max(1, INT64_HEADROOM // bound)
    return sum(int(np.dot(a[i:i + step], b[i:i + step])) for i in range(0, a.size, step))


def std_from_sums(s1, s2, n, eps):
    """_std_from_sums (stats.py:58-62)."""
    if n < 2:
        raise OracleError("ValueError", "standard deviation requires at least 2 points")
    num = s2 * n - s1 * s1
    return math.sqrt(num / (n * (n - 1))) * 2.0 * eps


def var_from_sums(s1, s2, n, eps):
    """N1 (not in reference): square of std_from_sums' radicand, scaled by (2*eps)^2."""
    if n < 2:
        raise OracleError("ValueError", "variance requires at least 2 points")
    num = s2 * n - s1 * s1
    return num / (n * (n - 1)) * ((2.0 * eps) * (2.0 * eps))


def mean_from_meta(metadata, sizes, eps):
    """stats.py:69-77."""
    n = int(np.asarray(sizes).sum())
    return exact_dot(metadata, sizes) / n * (2.0 * eps)


def lorenzo_weighted_sum(p, dims):
    """_lorenzo_weighted_sum (stats.py:95-112): sum(q) from Lorenzo residuals."""
    grid = np.asarray(p).reshape(dims)
    weights = [np.arange(n, 0, -1, dtype=np.int64) for n in dims]
    bound = grid.size and int(np.abs(grid).max())
    for w in weights:
        bound *= int(w[0])
    if bound < INT64_HEADROOM:
        spec = {2: "i,j,ij->", 3: "i,j,k,ijk->"}[len(dims)]
        return int(np.einsum(spec, *weights, grid.astype(np.int64)))
    total = 0
    for idx in np.ndindex(*dims[:-1]):
        row = int(np.dot(grid[idx].astype(np.int64), weights[-1]))
        for ax, i in enumerate(idx):
            row *= int(weights[ax][i])
        total += row
    return total


def mean_from_dp(c: Stream, p):
    """stats.py:80-92."""
    n = c.n
    if is_block_mean(c.kind):
        gd, gb = effective_geometry(c.kind, c.dims, c.block_dims)
        total = exact_sum(p) + exact_dot(c.metadata, block_sizes(gd, gb))
    elif c.kind == HSZP:
        total = exact_dot(p, np.arange(n, 0, -1, dtype=np.int64))
    else:
        total = lorenzo_weighted_sum(p, c.dims)
    return total / n * (2.0 * float(c.eps))


def block_mean_dev_sums(c: Stream, p):
    """HSZX* stage-2 integer mean and squared-deviation sum (stats.py:130-136)."""
    n = c.n
    gd, gb = effective_geometry(c.kind, c.dims, c.block_dims)
    sizes = block_sizes(gd, gb)
    weighted = exact_dot(c.metadata, sizes)
    mu = (2 * weighted + n) // (2 * n)
    dev = p.astype(np.int64) + np.repeat(c.metadata.astype(np.int64), sizes) - mu
    return mu, exact_dot(dev, dev)


def std_from_dp(c: Stream, p):
    """stats.py:125-144 (prefix kinds reduce to exact sums of q)."""
    n = c.n
    if is_block_mean(c.kind):
        if n < 2:
            raise OracleError("ValueError", "standard deviation requires at least 2 points")
        _, dd = block_mean_dev_sums(c, p)
        return math.sqrt(dd / (n - 1)) * 2.0 * c.eps
    q = recorrelate(p, None, c.kind, c.dims, c.block_dims)
    return std_from_sums(exact_sum(q), exact_dot(q, q), n, c.eps)


def var_from_dp(c: Stream, p):
    """N1 at stage 2: HSZX* uses the biased block-mean form squared (stats.py:130-138)."""
    n = c.n
    if is_block_mean(c.kind):
        if n < 2:
            raise OracleError("ValueError", "variance requires at least 2 points")
        _, dd = block_mean_dev_sums(c, p)
        return dd / (n - 1) * ((2.0 * c.eps) * (2.0 * c.eps))
    q = recorrelate(p, None, c.kind, c.dims, c.block_dims)
    return var_from_sums(exact_sum(q), exact_dot(q, q), n, c.eps)


def mean_from_dq(q, eps):
    """stats.py:115-118."""
    return exact_sum(q) / q.size * (2.0 * eps)


def std_from_dq(q, eps):
    """stats.py:168-173."""
    v = q.ravel()
    return std_from_sums(exact_sum(v), exact_dot(v, v), v.size, eps)


def var_from_dq(q, eps):
    v = q.ravel()
    return var_from_sums(exact_sum(v), exact_dot(v, v), v.size, eps)


def compute_stat(c: Stream, op, stage):
    """compute_stat (stats.py:195-212) plus op='var' (N1)."""
    if stage == META:
        if op != "mean":
            raise OracleError("UnsupportedStageError", "needs stage >= decorrelated")
        gd, gb = effective_geometry(c.kind, c.dims, c.block_dims)
        return mean_from_meta(c.metadata, block_sizes(gd, gb), c.eps)
    p = stage2(c)
    if stage == DECORRELATED:
        return {"mean": mean_from_dp, "std": std_from_dp, "var": var_from_dp}[op](c, p)
    q = stage3(c, p)
    if stage == QUANTIZED:
        return {"mean": mean_from_dq, "std": std_from_dq, "var": var_from_dq}[op](q, c.eps)
    d = stage4(c, q)
    if op == "mean":
        return float(np.mean(d))
    if op == "std":
        return float(np.std(d, ddof=1))
    return float(np.var(d, ddof=1))


# ---------------------------------------------------------------------------
# Stencils (analytics/fields.py)


def axis_central_diff(values, axis):
    """_axis_central_diff (fields.py:34-44)."""
    out = np.zeros(values.shape, dtype=values.dtype)
    lo = [slice(None)] * values.ndim
    hi = [slice(None)] * values.ndim
    mid = [slice(None)] * values.ndim
    lo[axis] = slice(0, -2)
    hi[axis] = slice(2, None)
    mid[axis] = slice(1, -1)
    out[tuple(mid)] = values[tuple(hi)] - values[tuple(lo)]
    return out


def laplacian_stencil(values):
    """_laplacian_stencil (fields.py:47-60); evaluation order kept for float inputs."""
    ndim = values.ndim
    interior = tuple(slice(1, -1) for _ in range(ndim))
    acc = (-2 * ndim) * values[interior]
    for axis in range(ndim):
        lo = [slice(1, -1)] * ndim
        hi = [slice(1, -1)] * ndim
        lo[axis] = slice(0, -2)
        hi[axis] = slice(2, None)
        acc = acc + values[tuple(lo)] + values[tuple(hi)]
    out = np.zeros(values.shape, dtype=acc.dtype)
    out[interior] = acc
    return out


def derivative_q(q, eps):
    """derivative_from_dq (fields.py:67-72)."""
    v = q.astype(np.int64)
    return [axis_central_diff(v, ax) * eps for ax in range(v.ndim)]


def laplacian_q(q, eps):
    """laplacian_from_dq (fields.py:75-80)."""
    v = q.astype(np.int64)
    if v.ndim < 2:
        raise OracleError("ValueError", "Laplacian requires 2D or 3D data")
    return [laplacian_stencil(v) * (2.0 * eps)]


def derivative_f(d):
    """derivative_from_df (fields.py:83-86)."""
    v = np.asarray(d, dtype=np.float64)
    return [axis_central_diff(v, ax) / 2.0 for ax in range(v.ndim)]


def laplacian_f(d):
    """laplacian_from_df (fields.py:89-93)."""
    v = np.asarray(d, dtype=np.float64)
    if v.ndim < 2:
        raise OracleError("ValueError", "Laplacian requires 2D or 3D data")
    return [laplacian_stencil(v)]


def derivative_p(c: Stream, p):
    """derivative_from_dp (fields.py:108-136) — the stage-2 homomorphic form."""
    if not is_nd(c.kind):
        raise OracleError("UnsupportedStageError", "no multidimensional layout")
    dims = c.dims
    eps = c.eps
    if c.kind == HSZX_ND:
        pg = as_grid(p, c.kind, dims, c.block_dims).astype(np.int64)
        mean = metadata_grid(c.metadata, c.kind, dims, c.block_dims)
        return [(axis_central_diff(pg, ax) + axis_central_diff(mean, ax)) * eps for ax in range(len(dims))]
    pg = p.astype(np.int64).reshape(dims)
    comps = []
    for ax in range(len(dims)):
        sel_mid = [slice(None)] * len(dims)
        sel_hi = [slice(None)] * len(dims)
        sel_mid[ax] = slice(1, -1)
        sel_hi[ax] = slice(2, None)
        pair = pg[tuple(sel_mid)] + pg[tuple(sel_hi)]
        for other in range(len(dims)):
            if other != ax:
                pair = np.cumsum(pair, axis=other)
        out = np.zeros(dims, dtype=np.int64)
        out[tuple(sel_mid)] = pair
        comps.append(out * eps)
    return comps


def laplacian_p(c: Stream, p):
    """laplacian_from_dp (fields.py:139-168)."""
    if not is_nd(c.kind):
        raise OracleError("UnsupportedStageError", "no multidimensional layout")
    dims = c.dims
    scale = 2.0 * c.eps
    if c.kind == HSZX_ND:
        pg = as_grid(p, c.kind, dims, c.block_dims).astype(np.int64)
        mean = metadata_grid(c.metadata, c.kind, dims, c.block_dims)
        return [(laplacian_stencil(pg) + laplacian_stencil(mean)) * scale]
    pg = p.astype(np.int64).reshape(dims)
    ndim = len(dims)
    interior = tuple(slice(1, -1) for _ in range(ndim))
    acc = None
    for ax in range(ndim):
        pref = pg
        for other in range(ndim):
            if other != ax:
                pref = np.cumsum(pref, axis=other)
        hi = [slice(1, -1)] * ndim
        lo = [slice(1, -1)] * ndim
        hi[ax] = slice(2, None)
        lo[ax] = slice(1, -1)
        contrib = pref[tuple(hi)] - pref[tuple(lo)]
        acc = contrib if acc is None else acc + contrib
    out = np.zeros(dims, dtype=np.int64)
    out[interior] = acc
    return [out * scale]


def field_op(c: Stream, op, stage):
    """compute_field_op (fields.py:181-196)."""
    if stage == META:
        raise OracleError("UnsupportedStageError", "stencil operations need stage >= decorrelated")
    p = stage2(c)
    if stage == DECORRELATED:
        return {"derivative": derivative_p, "laplacian": laplacian_p}[op](c, p)
    q = stage3(c, p)
    if stage == QUANTIZED:
        return {"derivative": derivative_q, "laplacian": laplacian_q}[op](q, c.eps)
    d = stage4(c, q)
    return {"derivative": derivative_f, "laplacian": laplacian_f}[op](d)


def divergence(sources, stage):
    """divergence (fields.py:216-222): float64 sum in component order."""
    derivs = [field_op(c, "derivative", stage) for c in sources]
    out = derivs[0][0].copy()
    for ax in range(1, len(derivs)):
        out += derivs[ax][ax]
    return out


def curl(sources, stage):
    """curl (fields.py:225-236)."""
    derivs = [field_op(c, "derivative", stage) for c in sources]
    if len(derivs) == 2:
        u, v = derivs
        return [u[1] - v[0]]
    u, v, w = derivs
    return [w[1] - v[2], u[2] - w[0], v[0] - u[1]]


def streamed_derivative(c: Stream):
    """streamed_derivative (fields.py:243-272) == derivative_from_dq on the whole grid."""
    return derivative_q(stage3(c), c.eps)


# ---------------------------------------------------------------------------
# N2-N5: new operations (not in the reference; SURVEY.md §8(a) definitions)


def region_dims(dims, region):
    """Region tiling = grid.partition semantics with the extent clipped to the grid."""
    r = (region,) * len(dims) if np.isscalar(region) else tuple(region)
    return tuple(min(int(a), int(n)) for a, n in zip(r, dims))


def region_reduce(q, region):
    """Per-region exact S1 (int), S2 (int), qmin, qmax, size in row-major region order."""
    dims = q.shape
    rd = region_dims(dims, region)
    g = block_grid(dims, rd)
    s1 = np.zeros(g, dtype=object)
    s2 = np.zeros(g, dtype=object)
    qmin = np.zeros(g, dtype=np.int32)
    qmax = np.zeros(g, dtype=np.int32)
    size = np.zeros(g, dtype=np.int64)
    for b in np.ndindex(*g):
        sl = tuple(slice(i * r, min((i + 1) * r, n)) for i, r, n in zip(b, rd, dims))
        t = q[sl].astype(np.int64).ravel()
        s1[b] = exact_sum(t)
        s2[b] = exact_dot(t, t)
        qmin[b] = t.min()
        qmax[b] = t.max()
        size[b] = t.size
    return s1, s2, qmin, qmax, size


def region_stats(q, eps, region):
    """N2: per-region mean and sample variance (NaN where size < 2)."""
    s1, s2, _, _, size = region_reduce(q, region)
    mean = np.zeros(size.shape)
    var = np.zeros(size.shape)
    for b in np.ndindex(*size.shape):
        n = int(size[b])
        mean[b] = int(s1[b]) / n * (2.0 * eps)
        var[b] = (float("nan") if n < 2 else
                  (n * int(s2[b]) - int(s1[b]) ** 2) / (n * (n - 1)) * ((2.0 * eps) * (2.0 * eps)))
    return mean, var


def region_minmax(q, eps, region):
    """N3: per-region min/max of the indices and of the stage-4 values."""
    _, _, qmin, qmax, _ = region_reduce(q, region)
    return qmin, qmax, qmin.astype(np.float64) * (2.0 * eps), qmax.astype(np.float64) * (2.0 * eps)


def threshold_count(q, eps, region, tau):
    """N4: number of regions with min_r < tau <= max_r (fp64 comparisons)."""
    _, _, fmin, fmax = region_minmax(q, eps, region)
    return int(np.count_nonzero((fmin < tau) & (tau <= fmax)))


def gradient_magnitude(q, eps):
    """N5: eps * sqrt(sum_k D_k^2), D_k the integer central differences (0 off-stencil)."""
    v = q.astype(np.int64)
    ds = [axis_central_diff(v, ax) for ax in range(v.ndim)]
    if max(int(np.abs(d).max()) for d in ds) < 2**31:
        s = sum(d.astype(np.uint64) ** 2 for d in ds)
        return np.sqrt(s.astype(np.float64)) * eps
    s = sum(d.astype(object) ** 2 for d in ds)
    return np.sqrt(np.vectorize(float)(s)) * eps


# ---------------------------------------------------------------------------
# Float-domain textbook operators (hsz/oracle.py), shared with no homomorphic path


def oracle_stats(field):
    """oracle.py:14-21 (two-pass mean and sample std)."""
    d = np.asarray(field, dtype=np.float64).ravel()
    mu = d.sum() / d.size
    var = ((d - mu) ** 2).sum() / (d.size - 1)
    return float(mu), float(np.sqrt(var))


def _shift(d, axis, step):
    out = np.zeros_like(d)
    src = [slice(None)] * d.ndim
    dst = [slice(None)] * d.ndim
    if step > 0:
        src[axis] = slice(step, None)
        dst[axis] = slice(0, -step)
    else:
        src[axis] = slice(0, step)
        dst[axis] = slice(-step, None)
    out[tuple(dst)] = d[tuple(src)]
    return out


def _interior_mask(shape, axes):
    mask = np.ones(shape, dtype=bool)
    for ax in axes:
        edge = [slice(None)] * len(shape)
        edge[ax] = 0
        mask[tuple(edge)] = False
        edge[ax] = -1
        mask[tuple(edge)] = False
    return mask


def oracle_derivative(field, axis):
    """oracle.py:50-55."""
    d = np.asarray(field, dtype=np.float64)
    out = (_shift(d, axis, 1) - _shift(d, axis, -1)) / 2.0
    out[~_interior_mask(d.shape, [axis])] = 0.0
    return out


def oracle_laplacian(field):
    """oracle.py:58-66."""
    d = np.asarray(field, dtype=np.float64)
    acc = np.zeros_like(d)
    for ax in range(d.ndim):
        acc += _shift(d, ax, 1) + _shift(d, ax, -1)
    acc -= 2 * d.ndim * d
    acc[~_interior_mask(d.shape, range(d.ndim))] = 0.0
    return acc


def oracle_divergence(components):
    out = oracle_derivative(components[0], 0)
    for ax in range(1, len(components)):
        out = out + oracle_derivative(components[ax], ax)
    return out


def oracle_curl(components):
    if len(components) == 2:
        u, v = components
        return [oracle_derivative(u, 1) - oracle_derivative(v, 0)]
    u, v, w = components
    return [oracle_derivative(w, 1) - oracle_derivative(v, 2),
            oracle_derivative(u, 2) - oracle_derivative(w, 0),
            oracle_derivative(v, 0) - oracle_derivative(u, 1)]


# ---------------------------------------------------------------------------
# Test-field generators (tests/conftest.py:28-42 restated)


def random_field(rng, dims, kind="mixed"):
    if kind == "smooth":
        out = rng.normal(0, 0.05, size=dims)
        for ax in range(len(dims)):
            out = np.cumsum(out, axis=ax)
        out += rng.uniform(-2, 2)
    elif kind == "noise":
        out = rng.normal(rng.uniform(-3, 3), rng.uniform(0.1, 4), size=dims)
    else:
        a = random_field(rng, dims, "smooth")
        b = random_field(rng, dims, "noise")
        out = a + 0.25 * b
    return out.astype(np.float32)
