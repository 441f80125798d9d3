"""Full-size parity at BASELINE configs 2, 3 and 4 (the operations each config names), GPU vs oracle.

* config 2 — 100x500x500 (Gaussian-filtered noise, rel 1e-3), HSZP_ND and HSZX_ND: container bytes,
  stage 3, region mean / variance and min / max over 16^3 regions (N2, N3), gradient magnitude (N5);
* config 3 — 3 x 256x384x384 (k^-3 Gaussian random fields, rel 1e-3 per component), HSZP_ND and
  HSZX_ND: divergence at stages 2 and 3 (fields.py:216-222), Laplacian per component at stages 2 and 3
  (fields.py:47-80, 139-168), per-component mean (stats.py:80-118);
* config 4 — 512^3 log-normal (rel 1e-4, bit widths up to 13), all four kinds: container bytes,
  stages 2 and 3, region min / max over 8^3 regions, threshold-crossing counts at tau in {0.01, 1, 100}
  (N4) and the variance (N1) at stages 2 and 3.

Integers, containers and fp64 outputs bit-exact; fp32 outputs = fl32 of the oracle's fp64 values.
The oracle (oracle/hsz_oracle.py) is pinned to the reference by tests/test_oracle_golden.py; the
field generators are the SURVEY §8(d) synthetic stand-ins (paper_2603_25206_b200/synthetic.py).
"""

import numpy as np
import pytest

from oracle import hsz_oracle as O

pytestmark = pytest.mark.gpu


def _oracle_of(c):
    from paper_2603_25206_b200 import io

    return O.stream_from_bytes(io.stream_to_bytes(c))


@pytest.fixture(scope="module")
def H():
    import paper_2603_25206_b200 as h
    from paper_2603_25206_b200 import io
    from paper_2603_25206_b200.analytics import fields, regions, stats

    class NS:
        pass

    ns = NS()
    ns.h, ns.io, ns.fields, ns.regions, ns.stats = h, io, fields, regions, stats
    return ns


# ---- config 2 ---------------------------------------------------------------------------------


@pytest.fixture(scope="module")
def cfg2():
    from paper_2603_25206_b200 import synthetic

    return synthetic.config2_field()


@pytest.mark.parametrize("kind", [1, 3], ids=["hszp-nd", "hszx-nd"])
def test_config2_regions_gradmag(H, cfg2, kind):
    field = cfg2
    c = H.h.compress(field, H.h.CompressorKind(kind), H.h.ErrorBound("rel", 1e-3))
    ref = O.compress(field, kind, "rel", 1e-3)
    assert H.io.stream_to_bytes(c) == O.stream_to_bytes(ref)
    q = O.stage3(ref)
    assert np.array_equal(H.h.partial_decompress(c, H.h.Stage.QUANTIZED).values, q)
    R = 16
    s1, s2, qmin, qmax, size = O.region_reduce(q, R)
    mean, var = O.region_stats(q, c.eps, R)
    _, _, fmin, fmax = O.region_minmax(q, c.eps, R)
    for stage in (H.h.Stage.QUANTIZED, H.h.Stage.DECORRELATED):
        rs = H.regions.region_stats(c, R, stage)
        assert rs.grid == (7, 32, 32)
        assert np.array_equal(rs.s1, s1.astype(np.int64)) and np.array_equal(rs.size, size)
        assert all(int(a) == int(b) for a, b in zip(rs.s2.ravel(), s2.ravel()))
        assert np.array_equal(rs.qmin, qmin) and np.array_equal(rs.qmax, qmax)
        np.testing.assert_allclose(rs.mean, mean, rtol=1e-15, atol=0)
        np.testing.assert_allclose(rs.var, var, rtol=1e-12, atol=0)
        assert np.array_equal(rs.vmin, fmin) and np.array_equal(rs.vmax, fmax)
    g = H.regions.gradient_magnitude(c)
    want = O.gradient_magnitude(q, c.eps)
    assert np.array_equal(g, want)
    g32 = H.regions.gradient_magnitude(c, out_dtype=np.float32)
    assert np.array_equal(g32, want.astype(np.float32))


# ---- config 3 ---------------------------------------------------------------------------------


@pytest.fixture(scope="module")
def cfg3():
    from paper_2603_25206_b200 import synthetic

    return synthetic.config3_fields()


@pytest.mark.parametrize("kind", [1, 3], ids=["hszp-nd", "hszx-nd"])
def test_config3_divergence_laplacian_mean(H, cfg3, kind):
    cs = [H.h.compress(f, H.h.CompressorKind(kind), H.h.ErrorBound("rel", 1e-3)) for f in cfg3]
    refs = [_oracle_of(c) for c in cs]
    for st in (3, 2):
        stage = H.h.Stage(st)
        div = H.fields.divergence(cs, stage).components[0]
        want = O.divergence(refs, st)
        assert np.array_equal(div, want), st
        div32 = H.fields.divergence(cs, stage, out_dtype=np.float32).components[0]
        assert np.array_equal(div32, want.astype(np.float32)), st
    for c, ref in zip(cs, refs):
        q = O.stage3(ref)
        lap = O.laplacian_q(q, c.eps)[0]
        for st in (3, 2):
            got = H.fields.compute_field_op(c, "laplacian", H.h.Stage(st), out_dtype=np.float32).components[0]
            assert np.array_equal(got, lap.astype(np.float32)), st
            assert H.stats.compute_stat(c, "mean", H.h.Stage(st)).value == O.compute_stat(ref, "mean", st)


# ---- config 4 ---------------------------------------------------------------------------------


@pytest.fixture(scope="module")
def cfg4():
    from paper_2603_25206_b200 import synthetic

    return synthetic.config4_field()


@pytest.mark.parametrize("kind", [0, 1, 2, 3], ids=["hszp", "hszp-nd", "hszx", "hszx-nd"])
def test_config4_stages_regions_counts_variance(H, cfg4, kind):
    field = cfg4
    c = H.h.compress(field, H.h.CompressorKind(kind), H.h.ErrorBound("rel", 1e-4))
    ref = O.compress(field, kind, "rel", 1e-4)
    assert H.io.stream_to_bytes(c) == O.stream_to_bytes(ref)
    d = c.device().validate()
    assert d.desc.max_bitwidth >= 12               # the config's wide per-block bit widths
    p = O.stage2(ref)
    assert np.array_equal(H.h.partial_decompress(c, H.h.Stage.DECORRELATED).values, p)
    q = O.stage3(ref, p)
    assert np.array_equal(H.h.partial_decompress(c, H.h.Stage.QUANTIZED).values, q)
    want = {(3, "mean"): O.mean_from_dq(q, ref.eps), (3, "var"): O.var_from_dq(q, ref.eps),
            (3, "std"): O.std_from_dq(q, ref.eps), (2, "mean"): O.mean_from_dp(ref, p)}
    if kind in (0, 1):          # prefix kinds: stage-2 std / var are those of q (stats.py:125-165)
        want[(2, "var")], want[(2, "std")] = want[(3, "var")], want[(3, "std")]
    else:
        want[(2, "var")], want[(2, "std")] = O.var_from_dp(ref, p), O.std_from_dp(ref, p)
    for (st, op), w in want.items():
        assert H.stats.compute_stat(c, op, H.h.Stage(st)).value == w, (st, op)
    if kind in (1, 3):
        R = 8
        blocks = q.reshape(64, R, 64, R, 64, R)      # 512^3 tiles exactly into 8^3 regions (O.region_reduce)
        qmin, qmax = blocks.min(axis=(1, 3, 5)), blocks.max(axis=(1, 3, 5))
        fmin, fmax = qmin.astype(np.float64) * (2.0 * c.eps), qmax.astype(np.float64) * (2.0 * c.eps)
        gq = H.regions.region_minmax(c, R)
        assert np.array_equal(gq[0], qmin) and np.array_equal(gq[1], qmax)
        assert np.array_equal(gq[2], fmin) and np.array_equal(gq[3], fmax)
        for tau in (0.01, 1.0, 100.0):
            want = int(np.count_nonzero((fmin < tau) & (tau <= fmax)))
            assert H.regions.threshold_count(c, R, tau) == want, tau
