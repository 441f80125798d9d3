"""Exact fp32 by table (EM_TABLE, stencil.cuh) and the one-pass HSZX_ND API stencils (fields._fused_stencil).

* the table emitter (fl32(fl64(D * eps)) looked up for |D| < XT_R, the fp64 conversion chain otherwise) is
  bit-identical to the conversion emitter and to the oracle: smooth fields (every value from the table),
  rough fields (rows falling back to the chain), and |q| >= 2^27 (the pipeline redoes the pass with the
  conversion emitter);
* compute_field_op("derivative" / "laplacian") at stages 2 / 3 of 3-D HSZX_ND (8^3 blocks) with fp32 outputs
  runs hszg_fused_blocks with only the requested outputs; its results equal the oracle's float64 stencils
  rounded once to fp32 (fields.py:34-93), i.e. the reconstruct + K-STEN route bit for bit.
"""

import numpy as np
import pytest

from oracle import hsz_oracle as O

pytestmark = pytest.mark.gpu

DIMS = [(48, 24, 64), (48, 40, 136), (16, 8, 8)]


def _field(dims, case, seed=3):
    rng = np.random.default_rng(seed)
    f = O.random_field(rng, dims, "smooth")
    if case == "smooth":
        return f, 1e-3 * float(f.max() - f.min())
    if case == "rough":              # neighbour differences of thousands of eps: the table's fallback rows
        f = f + rng.normal(0.0, 1.0, size=dims).astype(np.float32) * float(f.max() - f.min())
        return f.astype(np.float32), 1e-4 * float(f.max() - f.min())
    if case == "offset":             # |q| ~ 2.5e8 > 2^27 from the block means, residuals of a few bits
        g = (1000.0 + 1e-3 * f).astype(np.float32)
        return g, 2e-6
    return f, 2e-9 * float(np.abs(f).max())      # "large": |q| up to ~2.5e8 > 2^27, wide residuals


def _oracle(field, kind, eps):
    c = O.compress(field, kind, "abs", eps, (8, 8, 8))
    q = O.stage3(c)
    return [o.astype(np.float32) for o in O.derivative_q(q, eps) + O.laplacian_q(q, eps)], q


@pytest.mark.parametrize("kind", [1, 3])
@pytest.mark.parametrize("case", ["smooth", "rough", "large"])
def test_pipeline_table_equals_conversion_emitter(kind, case):
    import torch

    from paper_2603_25206_b200 import pipeline

    dims = (48, 24, 64)
    f, eps = _field(dims, case)
    fd = torch.from_numpy(f).cuda()
    sf = pipeline.compress_shard(fd, kind, eps, (8, 8, 8), 0, dims[0], dims)
    want, q = _oracle(f, kind, eps)
    if case == "rough":
        d = np.abs(np.diff(q.astype(np.int64), axis=2))
        assert d.max() >= 2048 and (d < 2048).mean() > 0.1    # both table rows and fallback rows
    got = {}
    for table in (True, False):
        pipe = pipeline.WindowPipeline(sf, pipeline.Comm(), 16)
        pipeline.apply_settings(pipe, exact_fp32=True, exact_table=table, use_graph=True)
        assert pipe._emit_mode() == (pipeline.EM_TABLE if table else pipeline.EM_EXACT)
        outs = [torch.empty(dims, dtype=torch.float32, device="cuda") for _ in range(4)]
        res = pipe.run(outs)
        got[table] = [o.cpu().numpy() for o in outs]
        v = q.ravel()
        assert res["s1"] == O.exact_sum(v) and res["s2"] == O.exact_dot(v, v)
        assert pipe._emit_mode() == (pipeline.EM_TABLE if table else pipeline.EM_EXACT)   # redo restored
    for k in range(4):
        assert np.array_equal(got[True][k], want[k]), (case, k)
        assert np.array_equal(got[False][k], want[k]), (case, k)


@pytest.mark.parametrize("dims", DIMS, ids=lambda d: "x".join(map(str, d)))
@pytest.mark.parametrize("case", ["smooth", "rough", "offset", "large"])
def test_api_fused_stencil_hszx_nd(dims, case, monkeypatch):
    import torch

    import paper_2603_25206_b200 as h
    from paper_2603_25206_b200 import _lib
    from paper_2603_25206_b200.analytics import fields

    f, eps = _field(dims, case, seed=11)
    c = h.compress(f, h.CompressorKind.HSZX_ND, h.ErrorBound("abs", eps), block_dims=(8, 8, 8))
    want, q = _oracle(f, 3, c.eps)
    ds = c.device().validate()
    fused = ds.desc.max_bitwidth <= 16                   # the one-pass kernel's staging limit
    assert fused or case == "large"
    if case == "offset":
        assert np.abs(q).max() >= 2**27                  # the conversion emitter (mode 1) runs
    calls = []
    real = _lib.call

    def spy(name, *a, **k):
        calls.append(name)
        return real(name, *a, **k)

    monkeypatch.setattr(_lib, "call", spy)
    for stage in (h.Stage.DECORRELATED, h.Stage.QUANTIZED):
        calls.clear()
        d = fields.compute_field_op(c, "derivative", stage, out="torch", out_dtype=np.float32)
        assert ("hszg_fused_blocks" in calls) == fused and ("hszg_reconstruct" in calls) != fused
        for k in range(3):
            assert d.components[k].dtype == torch.float32
            assert np.array_equal(d.components[k].cpu().numpy(), want[k]), (stage, k)
        calls.clear()
        lap = fields.compute_field_op(c, "laplacian", stage, out="numpy", out_dtype=np.float32)
        assert ("hszg_fused_blocks" in calls) == fused
        assert np.array_equal(lap.components[0], want[3]), stage
    # float64 outputs keep the reconstruct + K-STEN route; rounding them once gives the fused fp32 values
    d64 = fields.compute_field_op(c, "derivative", h.Stage.QUANTIZED, out="numpy", out_dtype=np.float64)
    for k in range(3):
        assert np.array_equal(d64.components[k].astype(np.float32), want[k])


def test_fused_blocks_rejects_output_subsets_in_fast_mode():
    import ctypes

    import torch

    import paper_2603_25206_b200 as h
    from paper_2603_25206_b200 import _lib

    dims = (16, 8, 8)
    f, eps = _field(dims, "smooth")
    c = h.compress(f, h.CompressorKind.HSZX_ND, h.ErrorBound("abs", eps), block_dims=(8, 8, 8))
    ds = c.device().validate()
    o = torch.empty(dims, dtype=torch.float32, device="cuda")
    for mode, ptrs, ok in ((0, [o, o, o, None], False), (0, [None, None, None, o], False),
                           (2, [o, None, o, None], False), (2, [None, None, None, o], True)):
        err = _lib.Err()
        st = _lib.lib().hszg_fused_blocks(ctypes.byref(ds.geom), ctypes.byref(ds.desc), 0, dims[0], None, None,
                                          (ctypes.c_void_p * 4)(*[None if p is None else _lib.ptr(p) for p in ptrs]),
                                          None, 2, mode, _lib.stream_handle(), ctypes.byref(err))
        assert (st == 0) == ok, (mode, st, err.message)
    torch.cuda.synchronize()
