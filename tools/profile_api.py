"""Kernel breakdown of single API calls (torch.profiler / CUPTI) on a BASELINE config-4 field.

For each row: wall time of one warm call and the device time per kernel, so host overhead
(Python, ctypes, syncs) and the slow kernels separate.

    python tools/profile_api.py [--config 4]
"""

import argparse
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=4)
    args = ap.parse_args()
    import numpy as np
    import torch
    from torch.profiler import ProfilerActivity, profile

    import paper_2603_25206_b200 as h
    from paper_2603_25206_b200 import synthetic
    from paper_2603_25206_b200.analytics import fields, regions, stats
    from paper_2603_25206_b200.compressors import compress_device

    K, S = h.CompressorKind, h.Stage
    f = synthetic.config4_field() if args.config == 4 else synthetic.config3_fields()[0]
    fd = torch.from_numpy(f).cuda()
    for kind in (K.HSZP, K.HSZP_ND, K.HSZX, K.HSZX_ND):
        c = h.compress(f, kind, h.ErrorBound("rel", 1e-4))
        c.device()
        rows = {
            "var stage 2": lambda: stats.compute_stat(c, "var", S.DECORRELATED),
            "var stage 3": lambda: stats.compute_stat(c, "var", S.QUANTIZED),
            "compress": lambda: compress_device(fd, kind, c.eps, c.block_dims),
        }
        if kind.is_nd:
            rows["region stats R=8"] = lambda: regions.region_stats(c, 8)
            rows["threshold count"] = lambda: regions.threshold_count(c, 8, 1.0)
            rows["laplacian stage 3"] = lambda: fields.compute_field_op(c, "laplacian", S.QUANTIZED, out="torch",
                                                                        out_dtype=np.float32)
        for name, fn in rows.items():
            fn()
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            fn()
            torch.cuda.synchronize()
            wall = time.perf_counter() - t0
            with profile(activities=[ProfilerActivity.CUDA]) as prof:
                fn()
                torch.cuda.synchronize()
            ks = {}
            for e in prof.events():
                if e.device_type.name == "CUDA":
                    k = ks.setdefault(e.name[:60], [0, 0.0])
                    k[0] += 1
                    k[1] += e.device_time / 1e3
            dev = sum(v[1] for v in ks.values())
            print(f"{kind.name:8s} {name:20s} wall {wall * 1e3:7.3f} ms  device {dev:7.3f} ms", flush=True)
            for k, (n, t) in sorted(ks.items(), key=lambda kv: -kv[1][1])[:6]:
                print(f"      {t:8.3f} ms  x{n:<3d} {k}")


if __name__ == "__main__":
    main()
