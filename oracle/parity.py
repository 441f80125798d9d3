"""Plane-window parity checker (TEST INFRASTRUCTURE — used by tests/ and by bench.py's post-timed
parity probe only; never by the product package).

The windowed pipeline (paper_2603_25206_b200/pipeline.py) writes the 3-component gradient and the
Laplacian of a z-slab sharded field.  Its outputs for planes [a, b) depend only on q of planes
[a - 1, b + 1), so any plane window of a field too large for the CPU oracle is checked against the
reference definitions on a small slab:

* q of the slab comes either from the oracle's decode of the container's chunk range
  (`hsz_oracle.stage3` of a sub-stream) or from `hsz_oracle.quantize` of the field planes (the
  compressor is lossless in q: stage 3 of compress(f) == quantize(f), quant.py:69-82 /
  compressors.py:201-226 — pinned by the golden tests);
* the stencils are `hsz_oracle.derivative_q` / `laplacian_q` (fields.py:34-80) on that slab; planes
  whose z-neighbours lie outside the slab are dropped unless they are global boundary planes.
"""

from __future__ import annotations

import numpy as np

from . import hsz_oracle as O

# fast fp32 emitter: fl32(fl32(D) * fl32(eps)) vs fl32(D * eps) — at most 4 roundings of 2^-24
FAST_RTOL = 4 * 2.0 ** -24


def stencil_planes(q_slab, s: int, n0: int, eps: float):
    """Oracle (dz, dy, dx, lap) float64 for the planes of q_slab (global planes [s, s + len)) whose
    7-point neighbourhood is inside the slab or on the global boundary -> (z_lo, z_hi, outs)."""
    q = np.asarray(q_slab)
    e = s + q.shape[0]
    outs = O.derivative_q(q, eps) + O.laplacian_q(q, eps)
    lo = 0 if s == 0 else 1
    hi = q.shape[0] if e == n0 else q.shape[0] - 1
    return s + lo, s + hi, [o[lo:hi] for o in outs]


def compare(got, want, exact: bool) -> dict:
    """got: fp32 arrays, want: float64 oracle arrays (same shapes).  exact: got == fl32(want) bit for
    bit; fast: |got - want| <= FAST_RTOL |want| (and exact zeros where want is 0)."""
    n = 0
    worst = 0.0
    ok = True
    for g, w in zip(got, want):
        g = np.asarray(g)
        n += g.size
        if exact:
            ok &= bool(np.array_equal(g, w.astype(np.float32)))
        err = np.abs(g.astype(np.float64) - w)
        aw = np.abs(w)
        nz = aw > 0
        if np.any(err[~nz] != 0):
            ok = False
            worst = float("inf")
        if np.any(nz):
            rel = float((err[nz] / aw[nz]).max())
            worst = max(worst, rel)
            if not exact and rel > FAST_RTOL:
                ok = False
    return {"ok": ok, "values": int(n), "max_rel_err": worst}


def sub_stream(kind, dims, block_dims, eps, payload: bytes, offsets, metadata, c0: int, c1: int, m0=0, m1=0,
               nplanes=None):
    """The oracle Stream of chunks [c0, c1) of a container whose chunk range covers whole planes
    (HSZP_ND, from the first plane only: no Lorenzo carry) or whole block layers (HSZX_ND)."""
    offs = np.asarray(offsets, dtype=np.uint64)
    b0 = int(offs[c0])
    b1 = int(offs[c1]) if c1 < len(offs) else len(payload)
    sub_offs = (offs[c0:c1] - np.uint64(b0)).astype(np.uint64)
    sub_dims = (nplanes,) + tuple(dims[1:])
    bd = tuple(min(b, n) for b, n in zip(block_dims, sub_dims))
    meta = None if metadata is None else np.asarray(metadata)[m0:m1].copy()
    return O.Stream(kind, sub_dims, bd, eps, meta, sub_offs, bytes(payload[b0:b1]))


def leading_planes(c, nz: int):
    """The oracle Stream of the first nz planes (axis 0) of a 3-D container: a prefix of the chunk list
    (every kind's stream order covers whole leading planes: flat 1-D blocks, HSZP_ND planes, HSZX_ND
    block layers when nz is a multiple of the block depth) and of the block means.  Stage 2/3 of it
    equal the container's first nz planes (no carry: the prefixes start at plane 0)."""
    dims = tuple(c.dims)
    sub = (nz,) + dims[1:]
    n = int(np.prod(sub))
    spans = c.spans
    c1 = int(np.searchsorted(spans[:, 1], n)) + 1
    assert int(spans[c1 - 1, 1]) == n, "plane boundary is not a chunk boundary"
    offs = np.asarray(c.offsets, dtype=np.uint64)
    b1 = int(offs[c1]) if c1 < len(offs) else len(c.payload)
    bd = tuple(c.block_dims) if O.is_nd(c.kind) else (min(int(c.block_dims[0]), n),) + (1,) * (len(dims) - 1)
    bd = tuple(min(b, s) for b, s in zip(bd, sub)) if O.is_nd(c.kind) else bd
    meta = None
    if c.metadata is not None:
        gd, gb = O.effective_geometry(c.kind, sub, bd)
        meta = np.asarray(c.metadata)[:int(np.prod(O.block_grid(gd, gb)))].copy()
    return O.Stream(c.kind, sub, bd, c.eps, meta, offs[:c1].copy(), bytes(c.payload[:b1]))
