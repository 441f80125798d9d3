"""Parity of the EXACT configuration bench.py times (BASELINE configs[4] pipeline) against the oracle.

bench.py runs `WindowPipeline` with pipeline.HEADLINE_SETTINGS: CUDA-graph replay, W = 64 planes,
the HSZX_ND one-pass kernel (fused.cu), and for HSZP_ND the persistent side-stream band scans
(256-row bands, int8 band-local prefixes; int16 in the window of the field's first plane) under the
ring z-sweeps, with the fast fp32 emitter.  These tests run that configuration on n2 = 2048 rows of
the config-5 field itself (so the int8 prefixes hold as they do in the bench) and compare:

* every output value with the oracle (fields.py:34-80 on stage 3 of the oracle's own decode of the
  GPU container, compressors.py:201-226): bit-exact in exact mode, <= 4 * 2^-24 relative in fast mode;
* the exact global sums / mean / variance (stats.py:58-62, 115-118) bit for bit;
* a 2-rank run, emulated rank by rank, at n2 = 2048;
* a field beyond 2^32 elements (64-bit indexing): the top and bottom planes against the oracle
  and every plane of the two kinds against each other (both derive from the same q).
"""

import numpy as np
import pytest

from oracle import hsz_oracle as O
from oracle import parity as PAR

pytestmark = pytest.mark.gpu

DIMS = (72, 768, 2048)          # nz > W = 64: two windows, the second partial; 3 bands of 256 rows


def _headline_field(nz, n1, z0=0):
    """Planes [z0, z0+nz), rows [0, n1) of the 2048^3 config-5 field (device fp32)."""
    from paper_2603_25206_b200 import synthetic

    f = synthetic.gen_config5_slab(z0, z0 + nz, dims=(2048, 2048, 2048))
    return f[:, :n1].contiguous()


def _host_stream(ds, eps):
    meta = None if ds.metadata is None else ds.metadata.cpu().numpy()
    return O.Stream(ds.kind, ds.dims, ds.block_dims, eps, meta, ds.offsets.cpu().numpy().view(np.uint64),
                    ds.payload[:ds.payload_len].cpu().numpy().tobytes())


@pytest.fixture(scope="module")
def headline():
    import torch

    from paper_2603_25206_b200.quant import field_minmax

    fd = _headline_field(*DIMS[:2])
    lo, hi, _ = field_minmax(fd.reshape(-1))
    eps = 1e-3 * (hi - lo)
    torch.cuda.synchronize()
    return fd, eps


@pytest.fixture(scope="module")
def oracle_q(headline):
    """Stage 3 by the oracle from the oracle's own compression (== quantize(field), asserted)."""
    fd, eps = headline
    f = fd.cpu().numpy()
    return O.quantize(f, eps)


@pytest.mark.parametrize("kind", [1, 3], ids=["hszp-nd", "hszx-nd"])
@pytest.mark.parametrize("exact", [False, True], ids=["fast", "exact"])
def test_headline_config_vs_oracle(headline, oracle_q, kind, exact):
    import torch

    from paper_2603_25206_b200 import pipeline

    fd, eps = headline
    sf = pipeline.compress_shard(fd, kind, eps, (8, 8, 8), 0, DIMS[0], DIMS)
    pipe = pipeline.WindowPipeline(sf, pipeline.Comm(), 64)
    pipeline.apply_settings(pipe, **pipeline.HEADLINE_SETTINGS)
    pipe.band_rows_req = 256
    pipe.exact_fp32 = exact
    outs = [torch.empty(DIMS, dtype=torch.float32, device="cuda") for _ in range(4)]
    for _ in range(2):                       # first run captures the graph, second replays it
        res = pipe.run(outs)
    assert pipe._graph is not None
    if kind == 1:
        assert pipe.band_rows == 256 and pipe.overlap and pipe.l16 and pipe.l8, "not the bench's HSZP_ND path"
    else:
        assert pipe._one_pass_ok()
    # the oracle decodes the GPU's container itself
    q = O.stage3(_host_stream(sf.ds, eps))
    assert np.array_equal(q, oracle_q)
    want = O.derivative_q(q, eps) + O.laplacian_q(q, eps)
    for k, (g, w) in enumerate(zip(outs, want)):
        r = PAR.compare([g.cpu().numpy()], [w], exact)
        assert r["ok"], (k, r)
    v = q.ravel()
    s1, s2 = O.exact_sum(v), O.exact_dot(v, v)
    assert res["s1"] == s1 and res["s2"] == s2
    assert res["mean"] == O.mean_from_dq(q, eps) and res["var"] == O.var_from_dq(q, eps)
    assert res["vmin"] == int(v.min()) and res["vmax"] == int(v.max())


@pytest.mark.parametrize("kind", [1, 3], ids=["hszp-nd", "hszx-nd"])
def test_headline_config_two_ranks(headline, oracle_q, kind):
    """World 2 at n2 = 2048, emulated rank by rank (halo planes, HSZP_ND carry from slab totals)."""
    import torch

    from paper_2603_25206_b200 import pipeline

    fd, eps = headline
    world = 2
    ranks = []
    for r in range(world):
        z0, z1 = pipeline.shard_planes(DIMS[0], world, r, 16)
        lead = 1 if (kind == 1 and z0 > 0) else 0
        sf = pipeline.compress_shard(fd[z0 - lead:z1].contiguous(), kind, eps, (8, 8, 8), z0, z1, DIMS)
        p = pipeline.WindowPipeline(sf, pipeline.Comm(), 64)
        pipeline.apply_settings(p, **pipeline.HEADLINE_SETTINGS)
        p.band_rows_req = 256
        ranks.append(p)
    mine = [p.local_boundary(need_total=True) for p in ranks]
    Ts = [m["T"] for m in mine] if kind == 1 else None
    carries = [p.carry_from(Ts, r) for r, p in enumerate(ranks)]
    firsts = [p.finish_first(m, c) for p, m, c in zip(ranks, mine, carries)]
    to_lower = [f if f is not None else m["head"] for f, m in zip(firsts, mine)]
    to_upper = [m["tail"] for m in mine]
    q = oracle_q
    want = O.derivative_q(q, eps) + O.laplacian_q(q, eps)
    tot1 = tot2 = 0
    for r, p in enumerate(ranks):
        p.apply_boundary(carries[r], to_upper[r - 1] if r > 0 else None, to_lower[r + 1] if r < world - 1 else None)
        outs = [torch.empty((p.sf.nz,) + DIMS[1:], dtype=torch.float32, device="cuda") for _ in range(4)]
        part = p.run_prepared(outs)
        tot1 += part["s1"]
        tot2 += part["s2"]
        for k, (g, w) in enumerate(zip(outs, want)):
            res = PAR.compare([g.cpu().numpy()], [w[p.sf.z0:p.sf.z1]], False)
            assert res["ok"], (r, k, res)
    v = q.ravel()
    assert tot1 == O.exact_sum(v) and tot2 == O.exact_dot(v, v)


def _plane_checksums(t, step=32):
    """Per-plane int64 sums of the fp32 bit patterns (a checksum of checksums over the outputs)."""
    import torch

    sums = []
    for a in range(0, t.shape[0], step):
        sums.append(t[a:a + step].view(torch.int32).to(torch.int64).sum(dim=(1, 2)))
    return torch.cat(sums).cpu().numpy()


def test_headline_beyond_2p32_elements():
    """(1032, 2048, 2048) = 4.33e9 > 2^32 elements with the bench settings: the last planes (flat
    offsets > 2^32) and the first planes vs the oracle, every plane of HSZP_ND == HSZX_ND."""
    import torch

    from paper_2603_25206_b200 import pipeline
    from paper_2603_25206_b200.quant import field_minmax

    dims = (1032, 2048, 2048)
    assert int(np.prod(dims)) > 2**32
    fd = synthetic_slab(dims)
    lo, hi, _ = field_minmax(fd.reshape(-1))
    eps = 1e-3 * (hi - lo)
    checks = {"bottom": (0, 10), "top": (dims[0] - 10, dims[0])}
    host = {k: fd[a:b].cpu().numpy() for k, (a, b) in checks.items()}
    shards = {k: pipeline.compress_shard(fd, k, eps, (8, 8, 8), 0, dims[0], dims) for k in (1, 3)}
    del fd
    torch.cuda.empty_cache()
    outs = [torch.empty(dims, dtype=torch.float32, device="cuda") for _ in range(4)]
    sums = {}
    for k, sf in shards.items():
        pipe = pipeline.WindowPipeline(sf, pipeline.Comm(), 64)
        pipeline.apply_settings(pipe, **pipeline.HEADLINE_SETTINGS)
        res = pipe.run(outs)
        if k == 1:
            assert pipe.band_rows == 256 and pipe.l8
        for name, (a, b) in checks.items():
            za, zb, want = PAR.stencil_planes(O.quantize(host[name], eps), a, dims[0], eps)
            got = [o[za:zb].cpu().numpy() for o in outs]
            r = PAR.compare(got, want, False)
            assert r["ok"], (k, name, r)
        sums[k] = (res["s1"], res["s2"], [_plane_checksums(o) for o in outs])
        del pipe
    assert sums[1][0] == sums[3][0] and sums[1][1] == sums[3][1]
    for a, b in zip(sums[1][2], sums[3][2]):
        assert np.array_equal(a, b)


def synthetic_slab(dims):
    from paper_2603_25206_b200 import synthetic

    return synthetic.gen_config5_slab(0, dims[0], dims=(2048, 2048, 2048))[:, :dims[1]]
