"""ctypes binding of libhszg.so (include/hszg.h).

Torch is used only as the device allocator and for the current CUDA stream:
every tensor crosses the ABI as a plain device pointer (``uint64``).  The
library is loaded lazily; a missing ``.so`` or a missing CUDA device raises
``BackendUnavailableError`` — there is no CPU fallback by design.
"""

from __future__ import annotations

import ctypes
import os
import threading

import numpy as np

from .errors import (
    BackendUnavailableError,
    CorruptStreamError,
    EpsTooSmallError,
    HszError,
    UnsupportedStageError,
    ZeroValueRangeError,
)

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("HSZG_LIB") or os.path.join(HERE, "libhszg.so")   # HSZG_LIB: A/B builds

PAYLOAD_PAD = 16

OK, CORRUPT, EPS_TOO_SMALL, INVALID_ARG, UNSUPPORTED_STAGE, CUDA_ERR, ZERO_RANGE, VALUE = range(8)
I32, F32, F64 = 0, 1, 2
WS_VALIDATE, WS_RECONSTRUCT, WS_REDUCE, WS_ENCODE, WS_QUANTIZE, WS_QSUMS = range(6)
OP_DERIV, OP_LAPLACIAN, OP_GRADMAG, OP_DIVERGENCE, OP_CURL, OP_GRAD_LAP = range(6)


class Geom(ctypes.Structure):
    _fields_ = [
        ("kind", ctypes.c_int32),
        ("ndims", ctypes.c_int32),
        ("dims", ctypes.c_int64 * 3),
        ("block_dims", ctypes.c_int64 * 3),
        ("eps", ctypes.c_double),
        ("n", ctypes.c_int64),
        ("n_chunks", ctypes.c_int64),
        ("n_blocks", ctypes.c_int64),
        ("sdims", ctypes.c_int64 * 3),
        ("sblk", ctypes.c_int64 * 3),
        ("sgrid", ctypes.c_int64 * 3),
    ]


class StreamDesc(ctypes.Structure):
    _fields_ = [
        ("payload", ctypes.c_void_p),
        ("payload_len", ctypes.c_uint64),
        ("offsets", ctypes.c_void_p),
        ("metadata", ctypes.c_void_p),
        ("canonical", ctypes.c_int32),
        ("max_bitwidth", ctypes.c_int32),
    ]


class Err(ctypes.Structure):
    _fields_ = [
        ("status", ctypes.c_int32),
        ("detail", ctypes.c_int32),
        ("chunk", ctypes.c_int64),
        ("element", ctypes.c_int64),
        ("value", ctypes.c_int64),
        ("message", ctypes.c_char * 192),
    ]


class Sums(ctypes.Structure):
    _fields_ = [
        ("s1_lo", ctypes.c_uint64),
        ("s1_hi", ctypes.c_int64),
        ("s2_lo", ctypes.c_uint64),
        ("s2_hi", ctypes.c_int64),
        ("count", ctypes.c_int64),
        ("vmin", ctypes.c_int32),
        ("vmax", ctypes.c_int32),
        ("f1", ctypes.c_double),
        ("f2", ctypes.c_double),
    ]

    @property
    def s1(self) -> int:
        return (int(self.s1_hi) << 64) | int(self.s1_lo)

    @property
    def s2(self) -> int:
        return (int(self.s2_hi) << 64) | int(self.s2_lo)


SUMS_BYTES = ctypes.sizeof(Sums)
assert SUMS_BYTES == 64

_lock = threading.Lock()
_LIB = None

_P = ctypes.c_void_p
_I64 = ctypes.c_int64
_U64 = ctypes.c_uint64
_I32 = ctypes.c_int
_D = ctypes.c_double
_SZ = ctypes.c_size_t

# name -> argtypes (restype int unless noted)
_SIGS = {
    "hszg_geom_init": [ctypes.POINTER(Geom)],
    "hszg_locate_chunks": [ctypes.POINTER(Geom), _I64, _I64, _P, _P, _P],
    "hszg_validate": [ctypes.POINTER(Geom), ctypes.POINTER(StreamDesc), _P, _SZ, _P, ctypes.POINTER(Err)],
    "hszg_decode": [ctypes.POINTER(Geom), ctypes.POINTER(StreamDesc), _P, _P, ctypes.POINTER(Err)],
    "hszg_decode_spans": [_P, _U64, _P, _P, _P, _I64, _P, _P, _SZ, _P, ctypes.POINTER(Err)],
    "hszg_encode_spans_sizes": [_P, _P, _P, _I64, _P, _P, ctypes.POINTER(ctypes.c_uint64), _P, _SZ, _P,
                                ctypes.POINTER(Err)],
    "hszg_encode_spans_pack": [_P, _P, _P, _I64, _P, _P, _P, _P, ctypes.POINTER(Err)],
    "hszg_encode_sizes": [ctypes.POINTER(Geom), _P, _P, _P, ctypes.POINTER(ctypes.c_uint64), _P, _SZ, _P,
                          ctypes.POINTER(Err)],
    "hszg_encode_pack": [ctypes.POINTER(Geom), _P, _P, _P, _P, _P, ctypes.POINTER(Err)],
    "hszg_reconstruct": [ctypes.POINTER(Geom), ctypes.POINTER(StreamDesc), _P, _I32, _P, _SZ, _P,
                         ctypes.POINTER(Err)],
    "hszg_reconstruct_carry": [ctypes.POINTER(Geom), ctypes.POINTER(StreamDesc), _P, _I32, _P, _P, _SZ, _P,
                               ctypes.POINTER(Err)],
    "hszg_dequantize": [_P, _I64, _D, _P, _I32, _P],
    "hszg_recorrelate": [ctypes.POINTER(Geom), _P, _P, _P, _I32, _P, _SZ, _P, ctypes.POINTER(Err)],
    "hszg_add_plane": [_P, _P, _I64, _I64, _P],
    "hszg_plane_sum": [ctypes.POINTER(Geom), ctypes.POINTER(StreamDesc), _P, _P, ctypes.POINTER(Err)],
    "hszg_stream_perm": [ctypes.POINTER(Geom), _P, _P],
    "hszg_scatter_grid": [ctypes.POINTER(Geom), _P, _P, _I32, _P, _P],
    "hszg_metadata_grid": [ctypes.POINTER(Geom), _P, _P, _P],
    "hszg_quantized_sums": [ctypes.POINTER(Geom), ctypes.POINTER(StreamDesc), _P, _P, _SZ, _P,
                            ctypes.POINTER(Err)],
    "hszg_reduce_stream": [ctypes.POINTER(Geom), ctypes.POINTER(StreamDesc), _I32, _P, _P, _SZ, _P,
                           ctypes.POINTER(Err)],
    "hszg_reduce_array": [ctypes.POINTER(Geom), _P, _P, _I32, _P, _P, _SZ, _P],
    "hszg_reduce_i32": [_P, _I64, _P, _P, _SZ, _P],
    "hszg_reduce_f64": [_P, _I64, _D, _P, _P, _P, _SZ, _P],
    "hszg_reduce_dot": [_P, _P, _I64, _P, _P, _SZ, _P],
    "hszg_region_reduce": [_P, ctypes.c_int32, _P, _P, _P, _P, _P, _P, _P, _P, _P],
    "hszg_region_finalize": [_P, _P, _P, _P, _P, _P, _I64, _D, _D, _P, _P, _P, _P, _P, _P],
    "hszg_region_stream": [ctypes.POINTER(Geom), ctypes.POINTER(StreamDesc), _P, _P, _P, _P, _P, _P, _P, _P, _SZ, _P,
                           ctypes.POINTER(Err)],
    "hszg_reduce_flt": [_P, _I64, _P, _P, _P, _SZ, _P],
    "hszg_stencil": [_I32, ctypes.c_int32, _P, ctypes.c_int32, _P, _P, _I32, ctypes.c_int32, _P, _P],
    "hszg_stencil_window": [_I32, _P, ctypes.c_int32, _P, _P, _I32, ctypes.c_int32, _P, _I64, _I64, _I64, _I64, _P],
    "hszg_sums_combine": [_P, _I64, _P, _P],
    "hszg_minmax_f32": [_P, _I64, _P, _P, _P, _SZ, _P],
    "hszg_minmax_f64": [_P, _I64, _P, _P, _P, _SZ, _P],
    "hszg_quantize_f32": [_P, _I64, _D, _P, _P, _SZ, _P, ctypes.POINTER(Err)],
    "hszg_quantize_f64": [_P, _I64, _D, _P, _P, _SZ, _P, ctypes.POINTER(Err)],
    "hszg_decorrelate": [ctypes.POINTER(Geom), _P, _P, _P, _P, _SZ, _P, ctypes.POINTER(Err)],
    "hszg_decorrelate_sized": [ctypes.POINTER(Geom), _P, _P, _P, _P, _P, ctypes.POINTER(ctypes.c_int), _P, _SZ, _P,
                               ctypes.POINTER(Err)],
    "hszg_encode_offsets": [ctypes.POINTER(Geom), _P, ctypes.POINTER(ctypes.c_uint64), _P, _SZ, _P,
                            ctypes.POINTER(Err)],
    "hszg_compress_plan": [ctypes.POINTER(Geom), ctypes.POINTER(ctypes.c_uint64), ctypes.POINTER(ctypes.c_uint64)],
    "hszg_compress_fused": [ctypes.POINTER(Geom), _P, _D, _P, ctypes.c_uint64, _P, _P, ctypes.POINTER(ctypes.c_uint64),
                            _P, _SZ, _P, ctypes.POINTER(Err)],
    "hszg_acc_reset": [_P, _P],
    "hszg_zgrad_lap": [_P, _I64, _I64, _I64, _I64, _I64, _I64, _D, _P, _P, _P, _P, _I32, _P],
    "hszg_zsweep_grad_lap": [_P, _I64, _I64, _I64, _P, _P, _P, _P, _I64, _I64, _D, _P, _P, _P, _P, _I64, _I32, _I32,
                             _P],
    "hszg_fused_blocks": [ctypes.POINTER(Geom), ctypes.POINTER(StreamDesc), _I64, _I64, _P, _P, _P, _P, _I64, _I32,
                          _P, ctypes.POINTER(Err)],
    "hszg_lorenzo_onepass": [ctypes.POINTER(Geom), ctypes.POINTER(StreamDesc), _P, _P, _P, _P, _I64, _I64, _P, _P,
                             _I32, _P, ctypes.POINTER(Err)],
    "hszg_band_scan": [ctypes.POINTER(Geom), ctypes.POINTER(StreamDesc), _I64, _P, _P, _P, _I32, _P, _I32, _P,
                       ctypes.POINTER(Err)],
    "hszg_decode_rowscan": [ctypes.POINTER(Geom), ctypes.POINTER(StreamDesc), _P, _P, ctypes.POINTER(Err)],
    "hszg_col_scan": [_P, _I64, _I64, _I64, _P],
    "hszg_gen_noise": [_P, _I64, _I64, _P, ctypes.c_uint64, _P],
    "hszg_gauss_pass": [_P, _P, _I64, _I64, _P, _I32, _P, _I32, _P],
    "hszg_gauss_pass_z": [_P, _P, _I64, _I64, _I64, _I64, _P, _P, _I32, _P],
    "hszg_gen_modes": [_P, _I64, _I64, _P, _P, _I32, _D, _P],
}

EXPORTED_SYMBOLS = tuple(_SIGS) + ("hszg_workspace_bytes", "hszg_version")


def load_library(path: str = LIB_PATH) -> ctypes.CDLL:
    """Load libhszg.so and declare every C-ABI entry point (no device needed)."""
    if not os.path.exists(path):
        raise BackendUnavailableError(
            f"{path} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'`"
        )
    lib = ctypes.CDLL(path)
    for name, args in _SIGS.items():
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = ctypes.c_int
    lib.hszg_workspace_bytes.argtypes = [ctypes.POINTER(Geom), ctypes.POINTER(StreamDesc), _I32, _I32]
    lib.hszg_workspace_bytes.restype = ctypes.c_size_t
    lib.hszg_version.argtypes = []
    lib.hszg_version.restype = ctypes.c_char_p
    return lib


def lib() -> ctypes.CDLL:
    """The loaded library; requires a CUDA device (the product path is GPU-only)."""
    global _LIB
    if _LIB is None:
        with _lock:
            if _LIB is None:
                import torch

                if not torch.cuda.is_available():
                    raise BackendUnavailableError(
                        "no CUDA device: the HSZ hot path runs only on the B200 kernels (no CPU fallback)"
                    )
                _LIB = load_library()
    return _LIB


def torch():
    import torch as _t

    return _t


_DEVICES: dict = {}


def device():
    lib()  # raises BackendUnavailableError when there is no CUDA device
    t = torch()
    idx = t.cuda.current_device()
    d = _DEVICES.get(idx)
    if d is None:
        d = _DEVICES[idx] = t.device("cuda", idx)
    return d


def stream_handle() -> int:
    """The current CUDA stream of the current device (raw handle; the fast path of
    torch.cuda.current_stream().cuda_stream, which costs ~15 us per call)."""
    t = torch()
    raw = getattr(t._C, "_cuda_getCurrentRawStream", None)
    if raw is not None:
        return int(raw(t.cuda.current_device()))
    return t.cuda.current_stream().cuda_stream


def ptr(t) -> int:
    return 0 if t is None else int(t.data_ptr())


# ---------------------------------------------------------------------------
# workspace: one growing device buffer per (device, stream) — kernels on one stream use it in order,
# callers on different streams (threads) get different buffers

_WS: dict = {}


def workspace(nbytes: int):
    t = torch()
    key = (t.cuda.current_device(), stream_handle())
    buf = _WS.get(key)
    nbytes = max(int(nbytes), 256)
    if buf is None or buf.numel() < nbytes:
        _WS[key] = None
        if buf is not None:
            del buf
        buf = t.empty(nbytes, dtype=t.uint8, device=device())
        _WS[key] = buf
    return buf


def release_workspace():
    _WS.clear()


# ---------------------------------------------------------------------------
# errors

_EXC = {
    CORRUPT: CorruptStreamError,
    EPS_TOO_SMALL: EpsTooSmallError,
    INVALID_ARG: ValueError,
    UNSUPPORTED_STAGE: UnsupportedStageError,
    ZERO_RANGE: ZeroValueRangeError,
    VALUE: ValueError,
    CUDA_ERR: RuntimeError,
}


def raise_for(status: int, err: Err | None = None, what: str = ""):
    if status == OK:
        return
    msg = err.message.decode(errors="replace") if err is not None and err.message else ""
    if not msg:
        msg = f"{what}: libhszg status {status}"
    cls = _EXC.get(status, HszError)
    raise cls(msg)


_SYNC = os.environ.get("HSZG_SYNC") == "1"     # debugging: synchronise after every entry point


def call(fn_name: str, *args, err: Err | None = None):
    status = getattr(lib(), fn_name)(*args)
    raise_for(status, err, fn_name)
    if _SYNC and not torch().cuda.is_current_stream_capturing():
        try:
            torch().cuda.synchronize()
        except Exception as e:  # noqa: BLE001
            raise RuntimeError(f"{fn_name}: device fault after the call: {e}") from e


# ---------------------------------------------------------------------------
# geometry

def make_geom(kind: int, dims, block_dims, eps: float) -> Geom:
    g = Geom()
    g.kind = int(kind)
    g.ndims = len(dims)
    for i in range(3):
        g.dims[i] = int(dims[i]) if i < len(dims) else 1
        g.block_dims[i] = int(block_dims[i]) if i < len(block_dims) else 1
    g.eps = float(eps)
    status = load_geom_lib().hszg_geom_init(ctypes.byref(g))
    if status != OK:
        raise ValueError(f"invalid geometry kind={kind} dims={tuple(dims)} block_dims={tuple(block_dims)}")
    return g


_GEOM_LIB = None


def load_geom_lib():
    """Geometry setup is pure host code inside libhszg.so and needs no device."""
    global _GEOM_LIB
    if _LIB is not None:
        return _LIB
    if _GEOM_LIB is None:
        _GEOM_LIB = load_library()
    return _GEOM_LIB


def locate_chunks(g: Geom, first: int = 0, count: int | None = None):
    """Host-side closed-form chunk spans (no device): (starts, ends, segment ids)."""
    count = int(g.n_chunks) - first if count is None else count
    st = np.zeros(count, dtype=np.int64)
    en = np.zeros(count, dtype=np.int64)
    sg = np.zeros(count, dtype=np.int64)
    status = load_geom_lib().hszg_locate_chunks(ctypes.byref(g), first, count, st.ctypes.data, en.ctypes.data,
                                                sg.ctypes.data)
    raise_for(status, None, "hszg_locate_chunks")
    return st, en, sg


def ws_bytes(g: Geom, s: StreamDesc | None, op: int, out_type: int = I32) -> int:
    return int(lib().hszg_workspace_bytes(ctypes.byref(g), ctypes.byref(s) if s is not None else None, op, out_type))


def sums_tensor():
    """Device buffer for one HszgSums record (every producer writes all of it)."""
    t = torch()
    return t.empty(SUMS_BYTES, dtype=t.uint8, device=device())


_PINNED_SUMS = threading.local()      # per thread: the API stays reentrant across threads


def read_sums(buf) -> Sums:
    """HszgSums from a device buffer: one copy into a reused pinned record, then a stream sync."""
    t = torch()
    if buf.numel() != SUMS_BYTES or not buf.is_cuda:
        return Sums.from_buffer_copy(buf.cpu().numpy().tobytes())
    idx = buf.device.index
    cache = getattr(_PINNED_SUMS, "bufs", None)
    if cache is None:
        cache = _PINNED_SUMS.bufs = {}
    host = cache.get(idx)
    if host is None:
        host = cache[idx] = t.empty(SUMS_BYTES, dtype=t.uint8, pin_memory=True)
    host.copy_(buf, non_blocking=True)
    t.cuda.current_stream(buf.device).synchronize()
    return Sums.from_buffer_copy(host.numpy().tobytes())


def np_dtype_code(dtype) -> int:
    dtype = np.dtype(dtype)
    if dtype == np.int32:
        return I32
    if dtype == np.float32:
        return F32
    if dtype == np.float64:
        return F64
    raise ValueError(f"unsupported output dtype {dtype}")
