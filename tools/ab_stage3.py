"""A/B timing of the API stage-3 / stage-4 reconstruction on the BASELINE config-4 field (512^3):
median device time of one call over 20 repetitions, plus the per-kernel split of one call
(torch.profiler).  Env knobs (HSZG_RECON_BR, HSZG_STREAM, ...) are read by the library.

    HSZG_RECON_BR=128 python tools/ab_stage3.py --kinds 1
"""

import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--kinds", type=int, nargs="*", default=[0, 1, 2, 3])
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--stats", action="store_true", help="also time mean / variance at stages 2 and 3")
    args = ap.parse_args()
    import torch
    from torch.profiler import ProfilerActivity, profile

    import paper_2603_25206_b200 as h
    from paper_2603_25206_b200 import synthetic
    from paper_2603_25206_b200.analytics import stats

    f = synthetic.config4_field()
    S = h.Stage
    for kind in args.kinds:
        c = h.compress(f, h.CompressorKind(kind), h.ErrorBound("rel", 1e-4))
        c.device()
        calls = [(f"stage {int(st)}", (lambda st=st: h.partial_decompress(c, st, out="torch"))) for st in (S.QUANTIZED, S.FULL)]
        if args.stats:
            calls += [(f"{op}@{int(st)}", (lambda op=op, st=st: stats.compute_stat(c, op, st)))
                      for op in ("mean", "var") for st in (S.DECORRELATED, S.QUANTIZED)]
        for label, fn in calls:
            for _ in range(3):
                fn()
            torch.cuda.synchronize()
            ts = []
            for _ in range(args.reps):
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record()
                fn()
                b.record()
                torch.cuda.synchronize()
                ts.append(a.elapsed_time(b))
            ts.sort()
            with profile(activities=[ProfilerActivity.CUDA]) as prof:
                fn()
                torch.cuda.synchronize()
            ks = {}
            for e in prof.events():
                if e.device_type.name == "CUDA":
                    name = e.name.split("<")[0].split("(")[0][:40]
                    ks[name] = ks.get(name, 0.0) + e.device_time
            split = {k: round(v, 1) for k, v in sorted(ks.items(), key=lambda kv: -kv[1])[:5]}
            print(f"kind {kind} {label} BR={os.environ.get('HSZG_RECON_BR', '-')} "
                  f"median {ts[len(ts) // 2]:.3f} ms min {ts[0]:.3f}  {split}", flush=True)


if __name__ == "__main__":
    main()
