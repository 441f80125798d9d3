"""Probe: API stencils at stage 3 (reconstruct + k_stencil_v4) vs the one-pass pipeline kernels on one
whole field (config 4, 512^3), exact and fast fp32 emitters, all four outputs or a subset (null outputs).

    python tools/probe_api_fused.py [--dims 512 512 512]
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def med_ms(fn, reps=9):
    import torch
    fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    ts.sort()
    return ts[len(ts) // 2]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--dims", type=int, nargs=3, default=[512, 512, 512])
    args = ap.parse_args()
    import numpy as np
    import torch
    import paper_2603_25206_b200 as h
    from paper_2603_25206_b200 import synthetic, pipeline as P
    from paper_2603_25206_b200.analytics import fields
    S = h.Stage
    f = synthetic.config4_field(dims=tuple(args.dims))
    for kind in (h.CompressorKind.HSZX_ND, h.CompressorKind.HSZP_ND):
        c = h.compress(f, kind, h.ErrorBound("rel", 1e-4))
        d = c.device()
        n = c.shape.total
        algo_in = d.payload_len + 8 * d.n_chunks + (0 if d.metadata is None else 4 * d.metadata.numel())
        res = {}
        res["api_grad"] = med_ms(lambda: fields.compute_field_op(c, "derivative", S.QUANTIZED, out="torch",
                                                                 out_dtype=np.float32))
        res["api_lap"] = med_ms(lambda: fields.compute_field_op(c, "laplacian", S.QUANTIZED, out="torch",
                                                                out_dtype=np.float32))
        sf = P.ShardedField(int(kind), c.eps, tuple(c.shape.dims), tuple(c.block_dims), 0, c.shape.dims[0], d)
        outs = [torch.empty(tuple(c.shape.dims), dtype=torch.float32, device="cuda") for _ in range(4)]
        for exact in (True, False):
            for sel, name in (((0, 1, 2, 3), "all4"),):
                pipe = P.WindowPipeline(sf, window=64)
                P.apply_settings(pipe, **dict(P.HEADLINE_SETTINGS, exact_fp32=exact))
                o = [outs[i] if i in sel else None for i in range(4)]
                try:
                    res[f"pipe_{'exact' if exact else 'fast'}_{name}"] = med_ms(lambda: pipe.run(o))
                except Exception as e:   # noqa: BLE001
                    res[f"pipe_{'exact' if exact else 'fast'}_{name}"] = f"ERR {e}"[:120]
        gb = lambda ms, outb: round((algo_in + outb * n) / (ms * 1e-3) / 1e9, 1) if isinstance(ms, float) else ms
        print(kind.name, {k: (round(v, 3) if isinstance(v, float) else v) for k, v in res.items()})
        print("   GB/s algo:", {k: gb(v, 12 if "grad" in k else (4 if "lap" in k else 16)) for k, v in res.items()})


if __name__ == "__main__":
    main()
