"""Chunk-codec plugin boundary (reference hsz/_kernels/__init__.py:11-22).

The reference picks a compiled Cython backend or a numpy fallback at import.
This package has exactly one backend: the sm_100a kernels of libhszg.so,
reached through the C ABI (``hszg_encode_spans_*`` / ``hszg_decode_spans``).
The signatures are the reference's — host arrays in, host arrays out — so
this module is a drop-in for byte-level parity tests; the throughput path
keeps streams resident on the device instead (``device.DeviceStream``).
"""

from __future__ import annotations

import ctypes

import numpy as np

from .. import _lib

BACKEND = "cuda-sm100a"


def _dev_i64(a):
    t = _lib.torch()
    return t.from_numpy(np.ascontiguousarray(a, dtype=np.int64)).to(_lib.device())


def encode_stream(values, starts, ends):
    """Encode consecutive chunks; returns (payload bytes, uint64 offsets) (_bitpack.pyx:14-87)."""
    t = _lib.torch()
    vals64 = np.asarray(values).astype(np.int64, copy=False)
    if vals64.size and (vals64.min() < -(2**31) or vals64.max() > 2**31 - 1):
        raise ValueError("chunk values must fit in signed 32 bits")
    n_chunks = len(starts)
    if n_chunks == 0:
        return b"", np.zeros(0, dtype=np.uint64)
    v = t.from_numpy(np.ascontiguousarray(vals64.astype(np.int32))).to(_lib.device())
    st = _dev_i64(starts)
    en = _dev_i64(ends)
    offs = t.empty(n_chunks, dtype=t.int64, device=_lib.device())
    bws = t.empty(n_chunks, dtype=t.uint8, device=_lib.device())
    total = ctypes.c_uint64(0)
    err = _lib.Err()
    ws = _lib.workspace(16 + 64 + (n_chunks // 256 + 2) * 20 + 512)
    _lib.call("hszg_encode_spans_sizes", _lib.ptr(v), _lib.ptr(st), _lib.ptr(en), n_chunks, _lib.ptr(offs),
              _lib.ptr(bws), ctypes.byref(total), _lib.ptr(ws), ws.numel(), _lib.stream_handle(), ctypes.byref(err),
              err=err)
    payload = t.empty(int(total.value) + _lib.PAYLOAD_PAD, dtype=t.uint8, device=_lib.device())
    _lib.call("hszg_encode_spans_pack", _lib.ptr(v), _lib.ptr(st), _lib.ptr(en), n_chunks, _lib.ptr(offs),
              _lib.ptr(bws), _lib.ptr(payload), _lib.stream_handle(), ctypes.byref(err), err=err)
    out = payload[: int(total.value)].cpu().numpy().tobytes()
    return out, offs.cpu().numpy().view(np.uint64).copy()


def decode_stream(payload, starts, ends, offsets):
    """Decode chunks back to int32 values in stream order (_bitpack.pyx:90-144)."""
    t = _lib.torch()
    buf = bytes(payload)
    n_chunks = len(starts)
    n = int(ends[n_chunks - 1]) if n_chunks > 0 else 0
    if n_chunks == 0:
        return np.zeros(0, dtype=np.int32)
    out = t.zeros(max(n, 1), dtype=t.int32, device=_lib.device())
    pay = t.zeros(len(buf) + _lib.PAYLOAD_PAD, dtype=t.uint8, device=_lib.device())
    if buf:
        pay[: len(buf)].copy_(t.frombuffer(bytearray(buf), dtype=t.uint8))
    st = _dev_i64(starts)
    en = _dev_i64(ends)
    offs = t.from_numpy(np.ascontiguousarray(np.asarray(offsets, dtype=np.uint64)).view(np.int64).copy()).to(
        _lib.device())
    err = _lib.Err()
    ws = _lib.workspace(256)
    _lib.call("hszg_decode_spans", _lib.ptr(pay), len(buf), _lib.ptr(st), _lib.ptr(en), _lib.ptr(offs), n_chunks,
              _lib.ptr(out), _lib.ptr(ws), ws.numel(), _lib.stream_handle(), ctypes.byref(err), err=err)
    return out[:n].cpu().numpy()
