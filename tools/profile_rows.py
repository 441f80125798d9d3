"""One call of each config-4 (512^3) API row, for ncu captures of the API kernels.

    ncu --set full --clock-control none --import-source on -k regex:'k_(reduce|tile|band|col|stencil|region)' \
        -o gpurun_out/rows python tools/profile_rows.py

Every row runs once to warm (lazy device upload, validation, workspaces) inside an NVTX range
"warm/<row>", then once more inside "rows/<kind>/<row>" — capture with
``--nvtx --nvtx-include 'rows/'`` to skip the warm-up launches.
"""

import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=4)
    ap.add_argument("--kinds", nargs="*", default=["HSZP", "HSZP_ND", "HSZX", "HSZX_ND"])
    ap.add_argument("--only", nargs="*", default=None, help="row name substrings")
    args = ap.parse_args()
    import numpy as np
    import torch

    import paper_2603_25206_b200 as h
    from paper_2603_25206_b200 import synthetic
    from paper_2603_25206_b200.analytics import fields, regions, stats

    K, S = h.CompressorKind, h.Stage
    f = synthetic.config4_field() if args.config == 4 else synthetic.config3_fields()[0]
    bound = h.ErrorBound("rel", 1e-4 if args.config == 4 else 1e-3)
    for name in args.kinds:
        kind = K[name]
        c = h.compress(f, kind, bound)
        c.device()
        rows = {
            "stage2": lambda: h.partial_decompress(c, S.DECORRELATED, out="torch"),
            "stage3": lambda: h.partial_decompress(c, S.QUANTIZED, out="torch"),
            "mean2": lambda: stats.compute_stat(c, "mean", S.DECORRELATED),
            "var2": lambda: stats.compute_stat(c, "var", S.DECORRELATED),
            "var3": lambda: stats.compute_stat(c, "var", S.QUANTIZED),
        }
        if kind.is_nd:
            rows["grad3"] = lambda: fields.compute_field_op(c, "derivative", S.QUANTIZED, out="torch",
                                                            out_dtype=np.float32)
            rows["lap3"] = lambda: fields.compute_field_op(c, "laplacian", S.QUANTIZED, out="torch",
                                                           out_dtype=np.float32)
            rows["region8"] = lambda: regions.region_stats(c, 8)
            rows["count8"] = lambda: regions.threshold_count(c, 8, 1.0)
        for rname, fn in rows.items():
            if args.only and not any(s in rname for s in args.only):
                continue
            torch.cuda.nvtx.range_push(f"warm/{name}/{rname}")
            fn()
            torch.cuda.synchronize()
            torch.cuda.nvtx.range_pop()
            torch.cuda.nvtx.range_push(f"rows/{name}/{rname}")
            fn()
            torch.cuda.synchronize()
            torch.cuda.nvtx.range_pop()
        del c
        torch.cuda.empty_cache()
    print("profile_rows: done")


if __name__ == "__main__":
    main()
