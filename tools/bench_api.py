"""API-level measurement of the other SURVEY §8 rows on BASELINE configs 1-4 (one B200).

Each row is timed through the package's public API in device mode (out="torch" where the API
has it; scalar results are host values, so their D2H is inside the timing), warm, median of
REPS CUDA-event timings.  Throughput is GB/s of original fp32 (4 N / t); the roofline fraction
uses SURVEY §8(d)'s algorithmic bytes per value with this stream's measured P (payload), I (index)
and Mb (block means) against MEASURED_PEAKS hbm_gbs.  Synthetic inputs follow §8(d)'s generators
(`paper_2603_25206_b200.synthetic`), seeded.  With ``--cpu-configs 1 2`` (the CPU baseline leg) every row
of those configs is also timed once on the CPU oracle (the reference algorithm restated, oracle/, single thread) on the same
container: ``cpu_oracle_ms`` and ``speedup_vs_cpu`` (the CPU path timed beside it).

    python tools/bench_api.py [--configs 1 2 3 4] [--out profiles/r01_api_bench.json]
"""

import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

REPS = 21


def timed(fn, reps=REPS):
    import torch

    fn()
    torch.cuda.synchronize()
    times = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        times.append(a.elapsed_time(b) / 1e3)
    times.sort()
    return times[len(times) // 2]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", type=int, nargs="*", default=[1, 2, 3, 4])
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "r01_api_bench.json"))
    ap.add_argument("--cpu-configs", type=int, nargs="*", default=[],
                    help="CPU baseline leg (opt-in): also time the CPU oracle (the reference algorithm restated, "
                         "1 thread) on these configs, e.g. --cpu-configs 1 2")
    args = ap.parse_args()

    import numpy as np
    import torch

    import paper_2603_25206_b200 as h
    from paper_2603_25206_b200 import synthetic
    from paper_2603_25206_b200.analytics import fields, regions, stats
    from paper_2603_25206_b200.compressors import compress_device

    with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
        peak = float(json.load(f)["hbm_gbs"])
    K = h.CompressorKind
    S = h.Stage
    rows = []

    O = None
    if args.cpu_configs:                 # the CPU baseline leg only: the oracle is never the measured path
        from oracle import hsz_oracle as O

        O.set_threads(1)

    def record(cfg, kind, row, n, t, algo_per_value, note="", cpu=None):
        gbs = 4.0 * n / t / 1e9
        ach = algo_per_value * n / t / 1e9
        r = {"config": cfg, "kind": kind.name, "row": row, "ms": round(t * 1e3, 3),
             "gbs_fp32": round(gbs, 1), "algo_B_per_value": round(algo_per_value, 3),
             "achieved_gbs": round(ach, 1), "frac": round(ach / peak, 3), "note": note}
        extra = ""
        if cpu is not None and cfg in args.cpu_configs:
            t0 = time.perf_counter()
            cpu()
            tc = time.perf_counter() - t0
            r["cpu_oracle_ms"] = round(tc * 1e3, 2)
            r["speedup_vs_cpu"] = round(tc / t, 1)
            extra = f"  cpu {tc * 1e3:9.1f} ms (x{tc / t:.0f})"
        rows.append(r)
        print(f"cfg{cfg} {kind.name:8s} {row:28s} {t * 1e3:9.3f} ms  {gbs:8.1f} GB/s-fp32  "
              f"{ach:8.1f} GB/s algo ({ach / peak:5.3f}){extra}", flush=True)

    gens = {
        1: (lambda: [synthetic.config1_field()], ("abs", 1e-4), [K.HSZP, K.HSZP_ND, K.HSZX, K.HSZX_ND]),
        2: (lambda: [synthetic.config2_field()], ("rel", 1e-3), [K.HSZP_ND, K.HSZX_ND]),
        3: (lambda: synthetic.config3_fields(), ("rel", 1e-3), [K.HSZP_ND, K.HSZX_ND]),
        4: (lambda: [synthetic.config4_field()], ("rel", 1e-4), [K.HSZP, K.HSZP_ND, K.HSZX, K.HSZX_ND]),
    }
    for cfg in args.configs:
        t0 = time.time()
        fields_np = gens[cfg][0]()
        mode, bound = gens[cfg][1]
        print(f"# config {cfg}: {len(fields_np)} x {fields_np[0].shape} generated in {time.time() - t0:.1f} s",
              flush=True)
        for kind in gens[cfg][2]:
            cs = []
            for f in fields_np:
                if mode == "abs":
                    bnd = h.ErrorBound("abs", bound * float(f.max() - f.min()))
                else:
                    bnd = h.ErrorBound("rel", bound)
                cs.append(h.compress(f, kind, bnd))
            c = cs[0]
            n = c.shape.total
            from paper_2603_25206_b200 import io as hio

            oc = O.stream_from_bytes(hio.stream_to_bytes(c)) if cfg in args.cpu_configs else None
            q3 = {}

            def oq():
                if "q" not in q3:
                    q3["q"] = O.stage3(oc)
                return q3["q"]
            d = c.device()
            P = d.payload_len / n
            I = 8.0 * d.n_chunks / n
            Mb = 0.0 if d.metadata is None else 4.0 * d.metadata.numel() / n
            nd = len(c.shape.dims)
            fd = torch.from_numpy(fields_np[0]).cuda()
            # E1-E5: compress from a device field (quantize + decorrelate + encode)
            t = timed(lambda: compress_device(fd, kind, c.eps, c.block_dims))
            record(cfg, kind, "E compress (device field)", n, t, 4 + P + I + Mb,
                   cpu=lambda: O.compress(fields_np[0], int(kind), "abs", c.eps,
                                          c.block_dims if kind.is_nd else c.block_dims[0]))
            # A1 / A3-A5: stages 2, 3, 4
            t = timed(lambda: h.partial_decompress(c, S.DECORRELATED, out="torch"))
            record(cfg, kind, "A1 stage 2 (p)", n, t, P + I + 4, cpu=lambda: O.stage2(oc))
            t = timed(lambda: h.partial_decompress(c, S.QUANTIZED, out="torch"))
            record(cfg, kind, "A3 stage 3 (q)", n, t, P + I + Mb + 4, cpu=lambda: O.stage3(oc))
            t = timed(lambda: h.partial_decompress(c, S.FULL, out="torch", dtype=torch.float32))
            record(cfg, kind, "A5 stage 4 (fp32)", n, t, P + I + Mb + 4, cpu=lambda: O.stage4(oc))
            # A8-A12, N1: statistics from the bytes
            if kind.is_block_mean:
                t = timed(lambda: stats.compute_stat(c, "mean", S.META))
                record(cfg, kind, "A8 mean at stage 1", n, t, Mb, cpu=lambda: O.compute_stat(oc, "mean", 1))
            t = timed(lambda: stats.compute_stat(c, "mean", S.DECORRELATED))
            record(cfg, kind, "A9 mean at stage 2", n, t, P + I + Mb, cpu=lambda: O.compute_stat(oc, "mean", 2))
            for st, name in ((S.DECORRELATED, "stage 2"), (S.QUANTIZED, "stage 3")):
                t = timed(lambda: stats.compute_stat(c, "var", st))
                record(cfg, kind, f"N1 variance at {name}", n, t, P + I + Mb,
                       cpu=lambda: O.compute_stat(oc, "var", int(st)))
            # A13/A14 (+A15 at stage 2 for nd kinds)
            if kind in (K.HSZP_ND, K.HSZX_ND):
                t = timed(lambda: fields.compute_field_op(c, "derivative", S.QUANTIZED, out="torch",
                                                          out_dtype=np.float32))
                record(cfg, kind, "A13 gradient at stage 3", n, t, P + I + Mb + 4 * nd,
                       cpu=lambda: O.field_op(oc, "derivative", 3))
                t = timed(lambda: fields.compute_field_op(c, "laplacian", S.QUANTIZED, out="torch",
                                                          out_dtype=np.float32))
                record(cfg, kind, "A14 Laplacian at stage 3", n, t, P + I + Mb + 4,
                       cpu=lambda: O.field_op(oc, "laplacian", 3))
            if cfg == 3 and kind in (K.HSZP_ND, K.HSZX_ND):
                t = timed(lambda: fields.divergence(cs, S.QUANTIZED, out="torch", out_dtype=np.float32))
                record(cfg, kind, "A16 divergence (3 comps)", 3 * n, t, (3 * (P + I + Mb) + 4) / 3)
            if cfg == 4 and kind in (K.HSZP_ND, K.HSZX_ND):
                # A7 slab iteration (reference slab semantics: one plane / one block row per slab), the
                # container device-resident vs streamed from pinned host memory
                from paper_2603_25206_b200 import io as hio

                hc = hio.stream_from_bytes(hio.stream_to_bytes(c))

                def drain(src, **kw):
                    for _ in h.slab_iter(src, S.QUANTIZED, out="torch", **kw):
                        pass

                t = timed(lambda: drain(c), reps=3)
                record(cfg, kind, "A7 slab_iter stage 3 (resident)", n, t, P + I + Mb + 4)
                t = timed(lambda: drain(hc, from_host=True), reps=3)
                record(cfg, kind, "A7 slab_iter stage 3 (from host)", n, t, P + I + Mb + 4,
                       note="container streamed H2D in 256 MB units; includes the pinned staging copy")
                del hc
            if cfg in (2, 4) and kind in (K.HSZP_ND, K.HSZX_ND):
                R = 16 if cfg == 2 else 8
                t = timed(lambda: regions.region_stats(c, R))
                record(cfg, kind, f"N2/N3 region stats R={R}", n, t, P + I + Mb,
                       cpu=lambda: (O.region_stats(oq(), c.eps, R), O.region_minmax(oq(), c.eps, R)))
                if cfg == 4:
                    t = timed(lambda: regions.threshold_count(c, 8, 1.0))
                    record(cfg, kind, "N4 threshold count", n, t, P + I + Mb)
                if cfg == 2:
                    t = timed(lambda: regions.gradient_magnitude(c, S.QUANTIZED, out="torch", out_dtype=np.float32))
                    record(cfg, kind, "N5 gradient magnitude", n, t, P + I + Mb + 4,
                           cpu=lambda: O.gradient_magnitude(oq(), c.eps))
            del fd
            torch.cuda.empty_cache()
    os.makedirs(os.path.dirname(args.out), exist_ok=True)
    with open(args.out, "w") as f:
        json.dump({"peak_gbs": peak, "reps": REPS, "rows": rows}, f, indent=1)


if __name__ == "__main__":
    main()
