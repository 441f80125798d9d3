"""Small-shape driver for compute-sanitizer (memcheck / racecheck / synccheck), one tool per run:

    compute-sanitizer --tool racecheck --error-exitcode 9 python tools/sanitize_run.py

Covers the warp-specialised mbarrier / TMA kernels (fused.cu one-pass HSZX_ND, window.cu band
scans + zring.cu ring z-sweeps in both the inline and the persistent side-stream form, lorenzo.cu
one-pass HSZP_ND), the warp-private TMA tiles of the fused statistics / regions (wtiles.cuh), and
one call of every API stage / op per kind, each checked against the oracle so a silent race would
also show as a wrong answer.
"""

import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import numpy as np
    import torch

    import paper_2603_25206_b200 as h
    from oracle import hsz_oracle as O
    from paper_2603_25206_b200 import io as hio
    from paper_2603_25206_b200 import pipeline
    from paper_2603_25206_b200.analytics import fields, regions, stats

    rng = np.random.default_rng(5)
    dims = (24, 16, 64)
    f = O.random_field(rng, dims, "smooth")
    eps = 1e-3 * float(f.max() - f.min())
    fd = torch.from_numpy(f).cuda()
    q_ref = O.quantize(f, eps)
    want = [o.astype(np.float32) for o in O.derivative_q(q_ref, eps) + O.laplacian_q(q_ref, eps)]
    cases = [
        (3, dict(one_pass=True)),                                     # fused.cu
        (1, dict(one_pass=False, band_rows_req=16, overlap=False)),   # window.cu + zring.cu inline
        (1, dict(one_pass=False, band_rows_req=16, overlap=True)),    # persistent side-stream scans
        (1, dict(one_pass=True, lorenzo_one_pass=True)),              # lorenzo.cu
    ]
    for kind, kw in cases:
        sf = pipeline.compress_shard(fd, kind, eps, (8, 8, 8), 0, dims[0], dims)
        p = pipeline.WindowPipeline(sf, pipeline.Comm(), 8)
        pipeline.apply_settings(p, exact_fp32=True, **kw)
        outs = [torch.empty(dims, dtype=torch.float32, device="cuda") for _ in range(4)]
        p.run(outs)
        torch.cuda.synchronize()
        for g, w in zip(outs, want):
            assert np.array_equal(g.cpu().numpy(), w), (kind, kw)
        print("pipeline ok", kind, kw, flush=True)
    for kind in h.CompressorKind:
        c = h.compress(f, kind, h.ErrorBound("abs", eps))
        oc = O.stream_from_bytes(hio.stream_to_bytes(c))
        assert np.array_equal(h.partial_decompress(c, h.Stage.DECORRELATED).values, O.stage2(oc))
        assert np.array_equal(h.partial_decompress(c, h.Stage.QUANTIZED).values, O.stage3(oc))
        for st in (2, 3):
            for op in ("mean", "var"):
                assert stats.compute_stat(c, op, h.Stage(st)).value == O.compute_stat(oc, op, st)
        if kind.is_nd:
            rs = regions.region_stats(c, 8)
            _, _, qmin, qmax, _ = O.region_reduce(O.stage3(oc), 8)
            assert np.array_equal(rs.qmin, qmin) and np.array_equal(rs.qmax, qmax)
            d = fields.compute_field_op(c, "laplacian", h.Stage.QUANTIZED).components[0]
            assert np.array_equal(d, O.laplacian_q(O.stage3(oc), c.eps)[0])
        print("api ok", kind.name, flush=True)
    torch.cuda.synchronize()
    print("sanitize_run: done")


if __name__ == "__main__":
    main()
