"""K-STEN: the vectorised stencil kernel (k_stencil_v4, four x-points per thread) against the scalar
k_stencil (forced by a 4-byte-misaligned input, which the vector path refuses) and the oracle.

Both kernels follow the reference's per-point fp64 sequence (fields.py:34-93), so every op, stage
domain, output type and shape must agree bit for bit.
"""

import zlib

import numpy as np
import pytest

from oracle import hsz_oracle as O

pytestmark = pytest.mark.gpu

OPS = ["deriv", "lap", "gradmag", "div", "curl", "grad_lap"]
SHAPES = [(7, 9, 4), (5, 6, 8), (4, 11, 132), (3, 5, 520), (13, 4), (9, 36), (3, 1028)]


def _code(op):
    from paper_2603_25206_b200 import _lib

    return {"deriv": _lib.OP_DERIV, "lap": _lib.OP_LAPLACIAN, "gradmag": _lib.OP_GRADMAG,
            "div": _lib.OP_DIVERGENCE, "curl": _lib.OP_CURL, "grad_lap": _lib.OP_GRAD_LAP}[op]


def _misaligned(q):
    """Same values at a 4-byte-offset address (not 16-B aligned: the scalar kernel runs)."""
    import torch

    buf = torch.empty(q.numel() + 1, dtype=q.dtype, device=q.device)
    v = buf[1:].view(q.shape)
    v.copy_(q)
    return v


@pytest.mark.parametrize("shape", SHAPES, ids=lambda s: "x".join(map(str, s)))
@pytest.mark.parametrize("op", OPS)
@pytest.mark.parametrize("domain", [0, 1])
@pytest.mark.parametrize("dtype", ["float32", "float64"])
def test_vector_matches_scalar(shape, op, domain, dtype):
    import torch

    from paper_2603_25206_b200 import device as devmod

    rng = np.random.default_rng(zlib.crc32(repr((shape, op, domain, dtype)).encode()))
    nd = len(shape)
    ncomp = nd if op in ("div", "curl") else 1
    big = op == "gradmag" and domain == 0
    lim = 2**31 - 1 if big else 1 << 20                     # gradmag: |D| up to 2^32, D^2 sums > 2^64
    qs = [torch.from_numpy(rng.integers(-lim, lim, size=shape, dtype=np.int64).astype(np.int32)).cuda()
          for _ in range(ncomp)]
    eps = [float(rng.uniform(1e-4, 1e-2)) for _ in range(ncomp)]
    dt = getattr(torch, dtype)
    code = _code(op)
    fast = devmod.stencil(code, qs, eps, domain, dt)
    slow = devmod.stencil(code, [_misaligned(q) for q in qs], eps, domain, dt)
    assert len(fast) == len(slow)
    for k, (a, b) in enumerate(zip(fast, slow)):
        assert torch.equal(a, b), (op, k)
    if op in ("deriv", "lap") and domain == 0 and dtype == "float64":
        q = qs[0].cpu().numpy()
        want = O.derivative_q(q, eps[0]) if op == "deriv" else O.laplacian_q(q, eps[0])
        for a, w in zip(fast, want):
            assert np.array_equal(a.cpu().numpy(), w)


@pytest.mark.parametrize("n", [1, 7, 4096, 1 << 20, (1 << 20) + 13])
def test_reduce_i32_extreme_values(n):
    """K-STAT over int32 arrays with |q| near 2^31 (squares near 2^62, pair sums near 2^63): exact."""
    import torch

    from paper_2603_25206_b200 import _lib, device as devmod

    rng = np.random.default_rng(n)
    x = rng.integers(-2**31, 2**31, size=n, dtype=np.int64)
    x[: min(n, 8)] = -2**31
    x32 = x.astype(np.int32)
    s = _lib.read_sums(devmod.reduce_i32(torch.from_numpy(x32).cuda()))
    assert s.s1 == int(x.sum())
    assert s.s2 == sum(int(v) * int(v) for v in x.tolist())
    assert s.vmin == int(x.min()) and s.vmax == int(x.max()) and s.count == n


@pytest.mark.parametrize("kind,dims,scale", [(0, (8192,), 1.0), (0, (40, 64), 1e6), (1, (12, 10, 64), 1.0),
                                             (1, (20, 8, 96), 1e6), (1, (300, 3, 32), 1.0)])
def test_quantized_sums_fused_matches_materialised(kind, dims, scale):
    """hszg_quantized_sums (q reduced where it is formed) == reconstruct + exact reduce, including
    |q| near 2^31 (per-thread int128 squares)."""
    import paper_2603_25206_b200 as h
    from paper_2603_25206_b200 import _lib, device as devmod

    rng = np.random.default_rng(len(dims) * 10 + kind)
    f = (O.random_field(rng, dims, "smooth") * scale).astype(np.float32)
    eps = 1e-6 * float(f.max() - f.min()) if scale > 1 else 1e-3 * float(f.max() - f.min())
    c = h.compress(f, h.CompressorKind(kind), h.ErrorBound("abs", eps))
    d = c.device()
    fused = d.quantized_sums()
    assert fused is not None
    a = _lib.read_sums(fused)
    b = _lib.read_sums(devmod.reduce_i32(d.reconstruct()))
    assert (a.s1, a.s2, a.vmin, a.vmax, a.count) == (b.s1, b.s2, b.vmin, b.vmax, b.count)


def test_api_reentrant_across_threads():
    """Two threads, each on its own CUDA stream, run the statistics / stage-3 API concurrently on
    different streams: per-stream workspaces and per-thread read-back buffers keep them apart."""
    import threading

    import torch

    import paper_2603_25206_b200 as h
    from paper_2603_25206_b200.analytics import stats

    rng = np.random.default_rng(11)
    fields = [O.random_field(rng, (24, 40, 64), "smooth") for _ in range(2)]
    cs = [h.compress(f, h.CompressorKind(k), h.ErrorBound("rel", 1e-3)) for f, k in zip(fields, (1, 3))]
    want = [(stats.compute_stat(c, "var", h.Stage.QUANTIZED).value,
             h.partial_decompress(c, h.Stage.QUANTIZED).values.copy()) for c in cs]
    errors = []

    def work(i):
        try:
            with torch.cuda.stream(torch.cuda.Stream()):
                for _ in range(20):
                    v = stats.compute_stat(cs[i], "var", h.Stage.QUANTIZED).value
                    q = h.partial_decompress(cs[i], h.Stage.QUANTIZED).values
                    if v != want[i][0] or not np.array_equal(q, want[i][1]):
                        errors.append(i)
                        return
        except Exception as e:  # pragma: no cover - reported below
            errors.append(repr(e))

    th = [threading.Thread(target=work, args=(i,)) for i in range(2)]
    for x in th:
        x.start()
    for x in th:
        x.join()
    assert not errors, errors
