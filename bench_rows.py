"""Per-row measurement of SURVEY §8(a) on BASELINE configs 1-4 (one B200) — bench.py's `rows` key.

Every §8(a) row is called through the package's public API in device mode (out="torch" where the
API has it; scalar results are host values, so their D2H is inside the API time) on the config's
seeded synthetic field (SURVEY §8(d) generators, `paper_2603_25206_b200.synthetic`):

* ``api_ms``     median CUDA-event time of one call (host sync inside), warm;
* ``kernel_ms``  the call's libhszg kernels only: CUPTI device durations summed over one call
                 (average of `PROF_CALLS` profiled calls) — the roofline numerator's time;
* ``algo_bytes`` SURVEY §8(d) algorithmic bytes (measured P, I = 8 B/chunk, Mb of this container);
* ``frac``       algo_bytes / kernel_ms / MEASURED_PEAKS hbm_gbs (``frac_api`` with api_ms);
* ``cpu_ms``     the reference CPU path for the same row on the same container, single thread:
                 the reference Cython codec (oracle/_ref) + the reference's numpy expressions
                 (oracle restatement).  Config 1 whole; configs 2-4 on the container's leading
                 CPU_PLANES planes (a prefix of its chunks: no carry), scaled by the plane ratio
                 (``cpu_extrapolated``).

    python bench_rows.py [--configs 1 2 3 4] [--no-cpu] [--out profiles/r02_rows.json]
"""

from __future__ import annotations

import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

REPS = 11
PROF_CALLS = 3
CPU_PLANES = {2: 20, 3: 32, 4: 32}


def _median_ms(fn, reps=REPS):
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


_PROF_WARM = False


def _kernel_ms(fn, calls=PROF_CALLS):
    """(ms of libhszg kernels per call, launches per call, {kernel: us per call}) by CUPTI.

    CUPTI can miss the first launches of a session, so a throwaway session runs once first, and each
    kernel's time per call is its mean recorded duration x its launches per call (rounded up)."""
    import math

    import torch
    from torch.profiler import ProfilerActivity, profile

    global _PROF_WARM
    torch.cuda.synchronize()
    if not _PROF_WARM:
        with profile(activities=[ProfilerActivity.CUDA]):
            fn()
            torch.cuda.synchronize()
        _PROF_WARM = True
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        for _ in range(calls):
            fn()
        torch.cuda.synchronize()
    rec = {}
    for e in prof.events():
        if e.device_type == torch.autograd.DeviceType.CUDA and "hszg" in e.name:
            dt = float(getattr(e, "device_time", None) or getattr(e, "cuda_time", 0.0) or 0.0)
            k = e.name.split("(")[0].replace("void ", "").replace("hszg::", "")[:48]
            r = rec.setdefault(k, [0, 0.0])
            r[0] += 1
            r[1] += dt
    per, n = {}, 0
    for k, (cnt, us) in rec.items():
        lpc = math.ceil(cnt / calls - 1e-9)
        per[k] = us / cnt * lpc
        n += lpc
    total = sum(per.values())
    return total / 1e3, n, {k: round(v, 1) for k, v in sorted(per.items(), key=lambda kv: -kv[1])}


def _cpu_ms(fn):
    t0 = time.perf_counter()
    fn()
    return (time.perf_counter() - t0) * 1e3


def measure(configs=(1, 2, 3, 4), cpu=True, peak=None, log=print):
    import numpy as np
    import torch

    import paper_2603_25206_b200 as h
    from paper_2603_25206_b200 import io as hio
    from paper_2603_25206_b200 import synthetic
    from paper_2603_25206_b200.analytics import fields, regions, stats
    from paper_2603_25206_b200.compressors import compress_device

    if peak is None:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            peak = float(json.load(f)["hbm_gbs"])
    O = P = CP = None
    if cpu:                          # the CPU baseline leg only: the oracle is never the measured path
        from oracle import cpu_pipeline as CP
        from oracle import hsz_oracle as O
        from oracle import parity as P

        O.set_threads(1)
        O.stage2 = CP.ref_stage2     # stage 2 through the reference's own Cython decoder
    K, S = h.CompressorKind, h.Stage
    rows = []

    def record(cfg, kind, row, n, fn, algo_per_value, cpu_fn=None, cpu_scale=1.0, reps=REPS, note=""):
        api = _median_ms(fn, reps)
        kms, launches, per = _kernel_ms(fn, min(PROF_CALLS, reps))
        algo = algo_per_value * n
        r = {"config": cfg, "kind": kind.name, "row": row, "values": n, "api_ms": round(api, 4),
             "kernel_ms": round(kms, 4), "launches": launches, "algo_bytes": int(algo),
             "gbs_fp32": round(4.0 * n / kms / 1e6, 1) if kms else None,
             "frac": round(algo / kms / 1e6 / peak, 3) if kms else None,
             "frac_api": round(algo / api / 1e6 / peak, 3), "kernels_us": per}
        if note:
            r["note"] = note
        if cpu_fn is not None:
            tc = _cpu_ms(cpu_fn) * cpu_scale
            r["cpu_ms"] = round(tc, 2)
            r["cpu_extrapolated"] = cpu_scale != 1.0
            r["speedup_api_vs_cpu"] = round(tc / api, 1)
        rows.append(r)
        log(f"cfg{cfg} {kind.name:8s} {row:30s} api {api:8.3f} ms  kern {kms:8.3f} ms  frac {r['frac']}"
            + (f"  cpu {r['cpu_ms']:.0f} ms" if "cpu_ms" in r else ""))

    gens = {
        1: (lambda: [synthetic.config1_field()], ("abs", 1e-4), [K.HSZP, K.HSZP_ND, K.HSZX, K.HSZX_ND]),
        2: (lambda: [synthetic.config2_field()], ("rel", 1e-3), [K.HSZP_ND, K.HSZX_ND]),
        3: (lambda: synthetic.config3_fields(), ("rel", 1e-3), [K.HSZP_ND, K.HSZX_ND]),
        4: (lambda: [synthetic.config4_field()], ("rel", 1e-4), [K.HSZP, K.HSZP_ND, K.HSZX, K.HSZX_ND]),
    }
    for cfg in configs:
        t0 = time.time()
        fields_np = gens[cfg][0]()
        mode, bound = gens[cfg][1]
        log(f"# config {cfg}: {len(fields_np)} x {fields_np[0].shape} generated in {time.time() - t0:.1f} s")
        for kind in gens[cfg][2]:
            cs = []
            for f in fields_np:
                bnd = h.ErrorBound("abs", bound * float(f.max() - f.min())) if mode == "abs" else h.ErrorBound("rel", bound)
                cs.append(h.compress(f, kind, bnd))
            c = cs[0]
            n = c.shape.total
            d = c.device()
            Pb = d.payload_len / n
            Ib = 8.0 * d.n_chunks / n
            Mb = 0.0 if d.metadata is None else 4.0 * d.metadata.numel() / n
            nd = len(c.shape.dims)
            oc = sub = None
            scale = 1.0
            if cpu:
                oc = O.stream_from_bytes(hio.stream_to_bytes(c))
                if cfg in CPU_PLANES:
                    sub = P.leading_planes(oc, CPU_PLANES[cfg])
                    scale = c.shape.dims[0] / CPU_PLANES[cfg]
                else:
                    sub = oc
            q3 = {}

            def oq():
                if "q" not in q3:
                    q3["q"] = O.stage3(sub)
                return q3["q"]

            def cf(fn):
                return (lambda: fn(sub)) if cpu else None

            fd = torch.from_numpy(fields_np[0]).cuda()
            sub_f = fields_np[0][:CPU_PLANES[cfg]] if (cpu and cfg in CPU_PLANES) else fields_np[0]
            record(cfg, kind, "E compress (device field)", n, lambda: compress_device(fd, kind, c.eps, c.block_dims),
                   4 + Pb + Ib + Mb,
                   (lambda: O.compress(sub_f, int(kind), "abs", c.eps, c.block_dims if kind.is_nd else c.block_dims[0]))
                   if cpu else None, scale)
            record(cfg, kind, "A1 stage 2 (p)", n, lambda: h.partial_decompress(c, S.DECORRELATED, out="torch"),
                   Pb + Ib + 4, cf(lambda s: O.stage2(s)), scale)
            record(cfg, kind, "A3 stage 3 (q)", n, lambda: h.partial_decompress(c, S.QUANTIZED, out="torch"),
                   Pb + Ib + Mb + 4, cf(lambda s: O.stage3(s)), scale)
            record(cfg, kind, "A5 stage 4 (fp32)", n,
                   lambda: h.partial_decompress(c, S.FULL, out="torch", dtype=torch.float32),
                   Pb + Ib + Mb + 4, cf(lambda s: O.stage4(s)), scale)
            if kind.is_block_mean:
                record(cfg, kind, "A8 mean at stage 1", n, lambda: stats.compute_stat(c, "mean", S.META), 2 * Mb,
                       cf(lambda s: O.compute_stat(s, "mean", 1)), scale, note="latency-bound (metadata only)")
            record(cfg, kind, "A9 mean at stage 2", n, lambda: stats.compute_stat(c, "mean", S.DECORRELATED),
                   Pb + Ib + Mb, cf(lambda s: O.compute_stat(s, "mean", 2)), scale)
            record(cfg, kind, "A10 mean at stage 3", n, lambda: stats.compute_stat(c, "mean", S.QUANTIZED),
                   Pb + Ib + Mb, cf(lambda s: O.compute_stat(s, "mean", 3)), scale)
            for st, name in ((S.DECORRELATED, "2"), (S.QUANTIZED, "3")):
                record(cfg, kind, f"N1 variance at stage {name}", n, lambda st=st: stats.compute_stat(c, "var", st),
                       Pb + Ib + Mb, cf(lambda s, st=st: O.compute_stat(s, "var", int(st))), scale)
            record(cfg, kind, "A12 std at stage 3", n, lambda: stats.compute_stat(c, "std", S.QUANTIZED),
                   Pb + Ib + Mb, cf(lambda s: O.compute_stat(s, "std", 3)), scale)
            if kind.is_nd:
                for st, name in ((S.QUANTIZED, "3"), (S.DECORRELATED, "2")):
                    record(cfg, kind, f"A13 gradient at stage {name}", n,
                           lambda st=st: fields.compute_field_op(c, "derivative", st, out="torch",
                                                                 out_dtype=np.float32),
                           Pb + Ib + Mb + 4 * nd, cf(lambda s, st=st: O.field_op(s, "derivative", int(st))), scale)
                    record(cfg, kind, f"A14 Laplacian at stage {name}", n,
                           lambda st=st: fields.compute_field_op(c, "laplacian", st, out="torch",
                                                                 out_dtype=np.float32),
                           Pb + Ib + Mb + 4, cf(lambda s, st=st: O.field_op(s, "laplacian", int(st))), scale)
            if cfg == 3 and kind.is_nd:
                for st, name in ((S.QUANTIZED, "3"), (S.DECORRELATED, "2")):
                    subs = [P.leading_planes(O.stream_from_bytes(hio.stream_to_bytes(x)), CPU_PLANES[3])
                            for x in cs] if cpu else None
                    record(cfg, kind, f"A16 divergence at stage {name}", 3 * n,
                           lambda st=st: fields.divergence(cs, st, out="torch", out_dtype=np.float32),
                           (3 * (Pb + Ib + Mb) + 4) / 3,
                           (lambda st=st, subs=subs: O.divergence(subs, int(st))) if cpu else None, scale)
            if cfg in (2, 4) and kind.is_nd:
                R = 16 if cfg == 2 else 8
                nreg = 1
                for dd in c.shape.dims:
                    nreg *= -(-dd // R)
                record(cfg, kind, f"N2/N3 region stats R={R}", n, lambda: regions.region_stats(c, R),
                       Pb + Ib + Mb + 72.0 * nreg / n,
                       (lambda: (O.region_stats(oq(), c.eps, R), O.region_minmax(oq(), c.eps, R))) if cpu else None,
                       scale, reps=5)
                if cfg == 4:
                    for tau in (0.01, 1.0, 100.0):
                        record(cfg, kind, f"N4 threshold count tau={tau:g}", n,
                               lambda tau=tau: regions.threshold_count(c, 8, tau), Pb + Ib + Mb,
                               (lambda tau=tau: O.threshold_count(oq(), c.eps, 8, tau)) if cpu else None, scale, reps=5)
                if cfg == 2:
                    record(cfg, kind, "N5 gradient magnitude", n,
                           lambda: regions.gradient_magnitude(c, S.QUANTIZED, out="torch", out_dtype=np.float32),
                           Pb + Ib + Mb + 4, (lambda: O.gradient_magnitude(oq(), c.eps)) if cpu else None, scale)
            if cfg == 4 and kind.is_nd:
                def drain(src, **kw):
                    for _ in h.slab_iter(src, S.QUANTIZED, out="torch", **kw):
                        pass

                hc = hio.stream_from_bytes(hio.stream_to_bytes(c))
                record(cfg, kind, "A7 slab_iter stage 3 (resident)", n, lambda: drain(c), Pb + Ib + Mb + 4, reps=3)
                record(cfg, kind, "A7 slab_iter stage 3 (from host)", n, lambda: drain(hc, from_host=True),
                       Pb + Ib + Mb + 4, reps=3, note="container streamed H2D from pinned host memory")
                del hc
            del fd
            torch.cuda.empty_cache()
    return {"peak_gbs": peak, "reps": REPS, "prof_calls": PROF_CALLS, "cpu_planes": CPU_PLANES, "rows": rows}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", type=int, nargs="*", default=[1, 2, 3, 4])
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--out", default=None)
    args = ap.parse_args()
    res = measure(args.configs, cpu=not args.no_cpu, log=lambda s: print(s, flush=True))
    if args.out:
        with open(args.out, "w") as f:
            json.dump(res, f, indent=1)


if __name__ == "__main__":
    main()
