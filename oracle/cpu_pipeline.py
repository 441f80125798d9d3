"""ORACLE — test/baseline infrastructure only (see oracle/__init__.py).

The reference CPU path for the benchmark workload (BASELINE config 5 step:
global mean/variance sums + 3-component gradient + Laplacian of HSZP_ND and
HSZX_ND streams), restated with the oracle (C codec + numpy, following
stages.py / analytics/*.py) and spread over all host cores with a process
pool: the bounded sample is a set of independent (8, 256, 2048) sub-fields
(eight planes x one 256-row band of the 2048^2 plane), each decompressed and
analysed end to end by one worker.  Used only by bench.py's ``cpu_baseline``
leg and its ``--impl reference`` arm.
"""

from __future__ import annotations

import math
import os
import time
from concurrent.futures import ProcessPoolExecutor

import numpy as np

from . import hsz_oracle as O

_HASH_KEY_MUL = 0x632BE59BD9B4E019
_M64 = np.uint64(0xFFFFFFFFFFFFFFFF)

SUB_PLANES = 8
SUB_ROWS = 256


def _splitmix64(x):
    with np.errstate(over="ignore"):
        x = x + np.uint64(0x9E3779B97F4A7C15)
        x = (x ^ (x >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        x = (x ^ (x >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        return x ^ (x >> np.uint64(31))


def config5_sample_field(z0: int, nz: int, dims=(2048, 2048, 2048), seed: int = 5) -> np.ndarray:
    """Host restatement of the device config-5 generator for planes [z0, z0+nz).

    Same construction (counter-hash Gaussian noise, separable Gaussian sigma 2 with reflect
    boundaries, 64 sinusoid modes); the mode sum uses Im(Y_z X) as two real GEMMs per plane.
    Only last-ulp float differences from the device field remain (irrelevant for a timing sample).
    """
    from scipy.ndimage import correlate1d

    N0, N1, N2 = dims
    rng = np.random.default_rng(seed)
    mag = rng.integers(1, 17, size=(64, 3))
    sign = rng.choice([-1, 1], size=(64, 3))
    k = (mag * sign).astype(np.float64)
    amp = 1.0 / np.sqrt((k ** 2).sum(axis=1))
    phase = rng.uniform(0.0, 2.0 * np.pi, size=64)
    r = 8
    x = np.arange(-r, r + 1, dtype=np.float64)
    w = np.exp(-0.5 * (x / 2.0) ** 2)
    w /= w.sum()
    e0, e1 = max(0, z0 - r), min(N0, z0 + nz + r)
    with np.errstate(over="ignore"):
        key = _splitmix64(np.uint64((seed * _HASH_KEY_MUL + 12345) & 0xFFFFFFFFFFFFFFFF))
    out = np.zeros((nz, N1, N2), dtype=np.float32)
    noise = np.empty((e1 - e0, N1, N2), dtype=np.float32)
    for z in range(e0, e1):
        idx = np.arange(z * N1 * N2, (z + 1) * N1 * N2, dtype=np.uint64)
        h = _splitmix64(idx ^ key)
        u1 = ((h >> np.uint64(40)).astype(np.float64) + 1.0) / 16777217.0
        u2 = (h & np.uint64(0xFFFFFF)).astype(np.float64) / 16777216.0
        plane = (np.sqrt(-2.0 * np.log(u1)) * np.cos(2.0 * np.pi * u2)).reshape(N1, N2)
        plane = correlate1d(plane, w, axis=1, mode="reflect")
        noise[z - e0] = correlate1d(plane, w, axis=0, mode="reflect")
    scale = 0.01 / math.sqrt(float((w ** 2).sum()) ** 3)
    ey = np.exp(2j * np.pi * np.outer(k[:, 1], np.arange(N1)) / N1)          # (64, N1)
    ex = np.exp(2j * np.pi * np.outer(k[:, 2], np.arange(N2)) / N2)          # (64, N2)
    for zl in range(nz):
        z = z0 + zl
        acc = np.zeros((N1, N2))
        for kk in range(-r, r + 1):
            zz = z + kk
            zz = -zz - 1 if zz < 0 else (2 * N0 - zz - 1 if zz >= N0 else zz)
            acc += w[kk + r] * noise[zz - e0]
        cz = amp * np.exp(1j * (2 * np.pi * k[:, 0] * z / N0 + phase))      # (64,)
        y = (cz[:, None] * ey)                                               # (64, N1)
        modes = y.real.T @ ex.imag + y.imag.T @ ex.real                      # Im(Y^T X)
        out[zl] = (modes + scale * acc).astype(np.float32)
    return out


def bands(field: np.ndarray):
    """Split a (Z, N1, N2) field into (SUB_PLANES, SUB_ROWS, N2) sub-fields."""
    Z, N1, _ = field.shape
    return [np.ascontiguousarray(field[z:z + SUB_PLANES, y:y + SUB_ROWS])
            for z in range(0, Z - SUB_PLANES + 1, SUB_PLANES) for y in range(0, N1 - SUB_ROWS + 1, SUB_ROWS)]


_REF = None


def ref_codec():
    """The reference's own Cython chunk codec (_bitpack.pyx, compiled into oracle/_ref by
    oracle/build_ref.sh), or None when it was not built."""
    global _REF
    if _REF is None:
        import sys

        d = os.path.join(os.path.dirname(os.path.abspath(__file__)), "_ref")
        try:
            if d not in sys.path:
                sys.path.insert(0, d)
            import _bitpack  # noqa: PLC0415

            _REF = _bitpack
        except ImportError:
            _REF = False
    return _REF or None


def ref_stage2(c):
    """Stage 2 through the reference decoder when present (_bitpack.decode_stream, _bitpack.pyx:90-144;
    called as codec.decode_stream does, codec.py:114-121), else the oracle's C restatement."""
    bp = ref_codec()
    sp = c.spans
    if bp is None:
        return O.decode_stream(c.payload, sp, c.offsets)
    return bp.decode_stream(c.payload, np.ascontiguousarray(sp[:, 0], dtype=np.int64),
                            np.ascontiguousarray(sp[:, 1], dtype=np.int64),
                            np.ascontiguousarray(c.offsets, dtype=np.uint64))


def _analyse(blob: bytes):
    """One worker: decompress a container to q and run the step's analytics (reference semantics)."""
    c = O.stream_from_bytes(blob)
    q = O.stage3(c, ref_stage2(c))                             # decode + recorrelate (stages.py:76-83)
    v = q.ravel()
    s1, s2 = O.exact_sum(v), O.exact_dot(v, v)                 # stats.py:168-173 sums
    grads = O.derivative_q(q, c.eps)                           # fields.py:67-72
    lap = O.laplacian_q(q, c.eps)                              # fields.py:75-80
    return s1, s2, v.size, float(grads[0].ravel()[0] + lap[0].ravel()[0])


def _compress(args):
    f, kind, eps = args
    return O.stream_to_bytes(O.compress(f, kind, "abs", eps))


def make_sample(fields, kinds, eps, pool=None):
    """Oracle-compress every sub-field with every kind (global absolute eps)."""
    jobs = [(f, kind, eps) for f in fields for kind in kinds]
    if pool is None:
        return [_compress(j) for j in jobs]
    return list(pool.map(_compress, jobs))


def make_pool(workers: int):
    import multiprocessing as mp

    if workers <= 1:
        return None
    return ProcessPoolExecutor(max_workers=workers, mp_context=mp.get_context("fork"))


def run_sample(blobs, pool=None):
    """Process every container (on the pool's processes); returns (seconds, elements, results)."""
    t0 = time.perf_counter()
    if pool is None:
        res = [_analyse(b) for b in blobs]
    else:
        res = list(pool.map(_analyse, blobs))
    dt = time.perf_counter() - t0
    return dt, sum(r[2] for r in res), res


def host_cores() -> int:
    return len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else (os.cpu_count() or 1)


def sample_planes(cores: int) -> int:
    """Planes in the bounded sample: enough (8x256-row) sub-fields to give every core one per stream."""
    per_slab = 2048 // SUB_ROWS
    slabs = max(1, min(4, -(-cores // per_slab)))
    return slabs * SUB_PLANES
