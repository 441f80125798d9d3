#!/usr/bin/env python
"""bench.py — BASELINE.json headline workload on N B200s (one process per GPU).

Workload (BASELINE configs[4], the one quoted for 1/2/4/8 GPUs): a 2048^3 fp32
field (64 random 3-D sinusoid modes + Gaussian-smoothed noise, seed 5,
generated on the device), rel error bound 1e-3 with the global value range,
compressed as HSZP_ND and HSZX_ND and z-slab partitioned across the ranks
(strong scaling).  One step = for each of the two compressed streams: exact
global mean + variance (int128 sums, one all-gather) and the 3-component
central-difference gradient + 5/7-point Laplacian straight from the
compressed bytes (one int32 halo plane per neighbour, HSZP_ND Lorenzo carry
by one all-gather), outputs written as fp32 grids.

value      = 2 streams x 4 B x 2048^3 / step time   (GB/s of original fp32, whole job)
e2e        = the same work from pinned HOST containers (H2D + validate + pipeline + D2H of every output)
roofline   = the dominant op's SURVEY §8(d) algorithmic bytes (compressed bytes + 16 B/value of fp32 outputs;
             intermediates do not count) / its CUDA-event time vs MEASURED_PEAKS hbm_gbs; per-kernel
             times in roofline.kernels
cpu_baseline = the reference path (oracle restatement: C codec + numpy) on a bounded sample, all host cores

--impl reference runs that reference CPU path alone (rank 0) on a bounded sample of the same workload.
"""

from __future__ import annotations

import argparse
import json
import math
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "GB/s of original fp32 per decompress-stage+op, % of HBM roofline, 1/2/4/8 GPU"
KINDS = (1, 3)              # HSZP_ND, HSZX_ND
KIND_NAMES = {1: "hszp-nd", 3: "hszx-nd"}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--dims", type=int, nargs=3, default=[2048, 2048, 2048])
    ap.add_argument("--window", type=int, default=64, help="planes per window (HSZX_ND: multiple of 8)")
    ap.add_argument("--exact-fp32", action="store_true",
                    help="fp32 outputs = fl32 of the reference float64 (default: fast fp32, <= 2^-22 relative)")
    ap.add_argument("--band-rows", type=int, default=None,
                    help="HSZP_ND band height of the band scan (default: sized by the pipeline; multiples of 16)")
    ap.add_argument("--no-graph", action="store_true", help="launch the window loop eagerly instead of a CUDA graph")
    ap.add_argument("--no-one-pass", action="store_true", help="HSZX_ND: two-pass (decode, then stencil) windows")
    ap.add_argument("--hszp-one-pass", action="store_true", help="HSZP_ND: the one-pass kernel (lorenzo.cu)")
    ap.add_argument("--overlap", type=int, default=1,
                    help="HSZP_ND: band scans on a side stream under the z-sweeps (1, default) or in line (0)")
    ap.add_argument("--e2e-steps", type=int, default=1)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--cpu-planes", type=int, default=4, help="planes per CPU-sample sub-field")
    ap.add_argument("--detail", default=None, help="write the per-kernel breakdown JSON here")
    ap.add_argument("--under-ncu", action="store_true", help="skip the CUPTI launch count (ncu owns the profiler)")
    ap.add_argument("--no-parity", action="store_true", help="skip the post-timed oracle parity probe")
    ap.add_argument("--no-exact", action="store_true", help="skip the exact-fp32 timing after the headline")
    ap.add_argument("--cpu-seconds", type=float, default=10.0, help="CPU baseline: seconds of all-core work")
    ap.add_argument("--rows", type=int, nargs="*", default=[4],
                    help="BASELINE configs whose per-row SURVEY §8(a) table goes into the line's `rows` (N = 1)")
    return ap.parse_args()


# ---------------------------------------------------------------------------
# clocks (nvidia-smi sampled during the timed region)


class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.rows = []
        self._stop = threading.Event()
        self._t = None

    def _run(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                                      "--format=csv,noheader,nounits"], capture_output=True, text=True, timeout=5)
                if out.returncode == 0 and out.stdout.strip():
                    self.rows.append([x.strip() for x in out.stdout.strip().split(",")])
            except Exception:  # noqa: BLE001
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self):
        import statistics

        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"], "samples": 0}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = set()
        for r in self.rows:
            for nm, v in zip(names, r[4:8]):
                if v.strip().lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(self.rows)}


# ---------------------------------------------------------------------------
# helpers


def measured_peak():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            return float(json.load(fh)["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:  # noqa: BLE001
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


class EventTimer:
    """CUDA events around each launch group on the launching (current) stream.

    Events are 'external', so inside a captured CUDA graph they become event-record nodes: after
    each replay they hold that replay's times (the last timed step)."""

    def __init__(self):
        import torch

        self.torch = torch
        self.open = {}
        self.rec = {}

    def clear(self):
        self.open.clear()
        self.rec.clear()

    def begin(self, name):
        e = self.torch.cuda.Event(enable_timing=True, external=True)
        e.record()
        self.open[name] = e

    def end(self, name, algo_bytes):
        e = self.torch.cuda.Event(enable_timing=True, external=True)
        e.record()
        self.rec.setdefault(name, []).append((self.open.pop(name), e, algo_bytes))

    def summary(self):
        self.torch.cuda.synchronize()
        out = {}
        for name, lst in self.rec.items():
            ms = sum(a.elapsed_time(b) for a, b, _ in lst)
            nbytes = sum(x for _, _, x in lst)
            out[name] = {"launch_groups": len(lst), "ms": ms, "algo_bytes": nbytes,
                         "gbs": nbytes / (ms / 1e3) / 1e9 if ms > 0 else None}
        return out


def count_kernel_launches(fn):
    """Kernels launched by one call of fn, counted by CUPTI (torch.profiler); only libhszg kernels."""
    import torch
    from torch.profiler import ProfilerActivity, profile

    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA]):      # CUPTI warm-up: a fresh session can miss
        fn()                                                # the first launches (bench_rows._kernel_ms)
        torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        fn()
        torch.cuda.synchronize()
    n = 0
    names = {}
    for evt in prof.events():
        if evt.device_type == torch.autograd.DeviceType.CUDA and "hszg" in evt.name:
            n += 1
            key = evt.name.split("(")[0][:80]
            rec = names.setdefault(key, {"launches": 0, "us": 0.0})
            rec["launches"] += 1
            dt = getattr(evt, "device_time", None)
            if dt is None:
                dt = getattr(evt, "cuda_time", 0.0)
            rec["us"] += float(dt or 0.0)
    return n, names


# ---------------------------------------------------------------------------
# our arm


def run_ours(args):
    import numpy as np
    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}")
    # HSZG_DIST_BACKEND=gloo: plumbing check of the multi-rank path with ranks sharing one GPU
    # (host-staged collectives; the timing of such a run is meaningless and is not a bench value)
    backend = os.environ.get("HSZG_DIST_BACKEND", "nccl")
    local = local % max(1, torch.cuda.device_count()) if backend == "gloo" else local
    torch.cuda.set_device(local)
    if world > 1:
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
    from paper_2603_25206_b200 import _lib, pipeline, synthetic
    from paper_2603_25206_b200.device import DeviceStream
    from paper_2603_25206_b200.quant import field_minmax

    comm = pipeline.Comm()
    N0, N1, N2 = args.dims
    n_total = N0 * N1 * N2
    z0, z1 = pipeline.shard_planes(N0, world, rank, 16)
    nz = z1 - z0
    t_setup = time.time()

    # ---- input: this rank's planes (+ one lead plane for the HSZP_ND predictor) -----------------
    lead = 1 if z0 > 0 else 0
    field = synthetic.gen_config5_slab(z0 - lead, z1, dims=(N0, N1, N2))
    lo, hi, bad = field_minmax(field[lead:].reshape(-1))
    mm = torch.tensor([lo, -hi], dtype=torch.float64, device="cuda")
    comm.all_reduce(mm, "min")
    eps = 1e-3 * (float(-mm[1]) - float(mm[0]))          # rel 1e-3 of the GLOBAL range (quant.py:56-66)
    cpu_blobs = None
    if rank == 0 and world == 1 and not args.no_cpu:
        cpu_blobs = build_cpu_sample(field[lead:], eps)
    shards = {}
    for kind in KINDS:
        src = field if kind == 1 else field[lead:]
        shards[kind] = pipeline.compress_shard(src, kind, eps, (8, 8, 8), z0, z1, (N0, N1, N2))
    del field, src
    torch.cuda.empty_cache()
    for sh in shards.values():
        sh.ds.validate()
    outs = [torch.empty((nz, N1, N2), dtype=torch.float32, device="cuda") for _ in range(4)]
    pipes = {k: pipeline.WindowPipeline(shards[k], comm, args.window) for k in KINDS}
    for p in pipes.values():
        p._range_bytes(0, 1)            # fetch the plane-boundary offsets for the timers now, not when timed
        p.use_graph = not args.no_graph
        p.exact_fp32 = args.exact_fp32
        p.one_pass = not args.no_one_pass
        p.lorenzo_one_pass = args.hszp_one_pass
        if args.overlap is not None:
            p.overlap = bool(args.overlap)
        if args.band_rows:
            p.band_rows_req = args.band_rows
    container_bytes = {k: shards[k].ds.nbytes() for k in KINDS}
    setup_s = time.time() - t_setup

    results = {}
    # per-stream CUDA-event timers around each launch group; under graph replay they are event
    # nodes of the captured graph and hold the last timed step's times
    timers = {k: EventTimer() for k in KINDS}
    spans = {k: EventTimer() for k in KINDS}     # one op = its whole run (launch groups may overlap)
    comm_timers = {k: EventTimer() for k in KINDS}
    for k in KINDS:
        pipes[k].timer = timers[k]
        if world > 1:
            pipes[k].comm_timer = comm_timers[k]

    def step():
        for k in KINDS:
            spans[k].begin("op")
            results[k] = pipes[k].run(outs)
            spans[k].end("op", 0)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    if args.no_graph:
        for tm in timers.values():
            tm.clear()
    for tm in list(spans.values()) + list(comm_timers.values()):
        tm.clear()
    comm.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clocks:
        ev0 = torch.cuda.Event(enable_timing=True)
        ev1 = torch.cuda.Event(enable_timing=True)
        ev0.record()
        for _ in range(args.steps):
            step()
        ev1.record()
        torch.cuda.synchronize()
    comm.barrier()
    ms_local = ev0.elapsed_time(ev1) / args.steps
    tt = torch.tensor([ms_local], dtype=torch.float64, device="cuda")
    comm.all_reduce(tt, "max")
    ms = float(tt.item())
    value = len(KINDS) * 4.0 * n_total / (ms / 1e3) / 1e9
    recorded_steps = args.steps if args.no_graph else 1
    kern = {}
    for k in KINDS:
        for name, v in timers[k].summary().items():
            key = f"{name}:{KIND_NAMES[k]}"
            kern[key] = v
    span_ms = {k: spans[k].summary()["op"]["ms"] / args.steps for k in KINDS}   # before any further step()
    if args.under_ncu:
        launches_per_step, launch_names = 0, {}
    else:
        launches_per_step, launch_names = count_kernel_launches(step)

    # ---- roofline of the dominant operation ----------------------------------------------------------
    # algorithmic bytes of "gradient (3 comps) + Laplacian, fp32, from the container" are
    # the compressed bytes read once (payload + index + block means) + 16 B/value written; passes over
    # intermediates (HSZP_ND's band-local prefix L) do not count.  An op = every kernel of one stream's
    # step (HSZP_ND: band scans + ring z-sweeps; HSZX_ND: the one-pass kernel); the dominant op is the
    # slower one.  Per-kernel numbers (with their own bytes) stay in `kernels`.
    peak, peak_src = measured_peak()
    ops = {}
    for k in KINDS:
        name = KIND_NAMES[k]
        groups = [g for g in kern if g.endswith(":" + name)]
        op_ms = span_ms[k]                                      # span of the op's run, every timed step
        algo = container_bytes[k] + 16 * nz * N1 * N2
        ops[name] = {"ms": op_ms, "algo_bytes": algo, "groups": groups}
    dom = max(ops, key=lambda k: ops[k]["ms"])
    d = ops[dom]
    achieved = d["algo_bytes"] / (d["ms"] / 1e3) / 1e9
    roofline = {"bound": "hbm", "kernel": f"op:{dom} ({' + '.join(d['groups'])})", "achieved": round(achieved, 1),
                "peak": peak, "unit": "GB/s", "frac": round(achieved / peak, 4), "traffic": None,
                "peak_source": peak_src, "share_of_step": round(d["ms"] / ms, 4),
                "algo_bytes_per_launch": int(d["algo_bytes"]),
                "launch": "one step of the op (all its kernels; time = the op's span, its launch groups may "
                          "overlap on two streams)",
                "other_ops": {o: {"achieved": round(v["algo_bytes"] / (v["ms"] / 1e3) / 1e9, 1),
                                  "frac": round(v["algo_bytes"] / (v["ms"] / 1e3) / 1e9 / peak, 4),
                                  "ms": round(v["ms"], 3)} for o, v in ops.items() if o != dom},
                "kernels": {g: {"ms_per_step": round(v["ms"] / recorded_steps, 3),
                                "gbs_own_bytes": round(v["gbs"], 1)} for g, v in kern.items()}}
    prof = measured_traffic(dom, (N0, N1, N2), world, args.window)
    if prof is not None:
        roofline["traffic"] = prof["traffic_bytes_per_step"]
        roofline["traffic_source"] = prof["source"]

    comm_ms = {}
    if world > 1:
        for k in KINDS:
            for name, v in comm_timers[k].summary().items():
                comm_ms[f"{name}:{KIND_NAMES[k]}"] = round(v["ms"] / max(1, v["launch_groups"]), 3)
        cm = torch.tensor(list(comm_ms.values()) or [0.0], dtype=torch.float64, device="cuda")
        comm.all_reduce(cm, "max")
        comm_ms = dict(zip(comm_ms, [round(x, 3) for x in cm.cpu().tolist()]))

    # ---- exact-fp32 emitter: the same step timed (fp32 outputs = fl32 of the reference float64) ----------
    exact = None
    if not args.no_exact and not args.exact_fp32:
        exact = time_exact(args, pipes, outs, comm, step, n_total)

    # ---- parity probe vs the oracle (after the timed region; the checker is not timed) ------------------
    parity = None
    if not args.no_parity:
        parity = parity_probe(args, pipes, outs, comm, eps, (N0, N1, N2), z0, z1)

    # ---- e2e: host containers in, every output back to the host ------------------------------------------
    e2e = None
    if not args.no_e2e:
        e2e = run_e2e(args, shards, pipes, outs, comm, n_total)

    # ---- CPU baseline (rank 0, N = 1) ---------------------------------------------------------------
    cpu = cpu_baseline(cpu_blobs, args.cpu_seconds) if cpu_blobs else None

    # ---- per-row table (SURVEY §8(a) rows on configs 1-4; N = 1, after the headline's buffers are freed) --
    rows = None
    if world == 1 and args.rows:
        # in a child process: a CUPTI session there starts clean (this process's earlier profiler sessions
        # and graph replays made later sessions drop kernel records)
        import tempfile

        del outs, pipes, shards
        torch.cuda.empty_cache()
        with tempfile.NamedTemporaryFile(suffix=".json") as tf:
            cmd = [sys.executable, os.path.join(ROOT, "bench_rows.py"), "--configs", *map(str, args.rows),
                   "--out", tf.name] + (["--no-cpu"] if args.no_cpu else [])
            r = subprocess.run(cmd, stdout=sys.stderr, stderr=sys.stderr)
            if r.returncode == 0:
                with open(tf.name) as fh:
                    rows = json.load(fh)
            else:
                rows = {"error": f"bench_rows.py exited {r.returncode}"}

    if rank == 0:
        s = results
        line = {
            "metric": METRIC, "value": round(value, 2), "unit": "GB/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(ms, 3), "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "int32",
            "data": "synthetic: config-5 generator (64 random 3-D sinusoid modes + Gaussian-smoothed noise sigma 2, "
                    "seed 5) generated on the device",
            "config": {"workload": "config5: 2048^3 fp32, rel eb 1e-3, HSZP_ND + HSZX_ND streams; per step "
                                   "global mean+variance and 3-comp gradient + Laplacian (fp32 out) from the "
                                   "compressed bytes, z-slab sharded",
                       "dims": [N0, N1, N2], "kinds": [KIND_NAMES[k] for k in KINDS], "window_planes": args.window, "fp32_outputs": "exact" if args.exact_fp32 else "fast",
                       "eps": eps, "container_bytes_rank0": {KIND_NAMES[k]: container_bytes[k] for k in KINDS},
                       "l2": "working set >> 126 MB L2 (inputs 5-8 GB, outputs 137 GB per stream)",
                       "parallelism": f"z-slab x{world}", "setup_s": round(setup_s, 1)},
            "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e,
            "gpu_launches": launches_per_step * args.steps,
            "clocks": clocks.summary(),
            "stats_check": {KIND_NAMES[k]: {"mean": s[k]["mean"], "var": s[k]["var"]} for k in KINDS},
            "exact_fp32": exact, "parity": parity, "rows": rows,
        }
        if world > 1:
            line["comm_ms_per_step"] = comm_ms
            line["nccl"] = {"backend": comm.dist.get_backend() if comm.dist else None, "ranks": world}
        print(json.dumps(line), flush=True)
        if args.detail:
            with open(args.detail, "w") as fh:
                json.dump({"kernels": kern, "launch_names": launch_names, "launches_per_step": launches_per_step,
                           "line": line}, fh, indent=1)
    if world > 1:
        dist.destroy_process_group()


def run_e2e(args, shards, pipes, outs, comm, n_total):
    """Containers from pinned host memory each step (+validation), outputs copied back to the host."""
    import torch

    host = {}
    for k, sh in shards.items():
        ds = sh.ds
        host[k] = (ds.payload.cpu().pin_memory(), ds.offsets.cpu().pin_memory(),
                   None if ds.metadata is None else ds.metadata.cpu().pin_memory())
    stage = torch.empty(64 * 1024 * 1024, dtype=torch.float32).pin_memory()   # 256 MB staging
    h2d = sum(sum(x.numel() * x.element_size() for x in host[k] if x is not None) for k in host)
    d2h = 0

    def e2e_step(copy_outputs=True):
        nonlocal d2h
        moved = 0
        for k, sh in shards.items():
            ds = sh.ds
            p, o, m = host[k]
            ds.payload.copy_(p, non_blocking=True)
            ds.offsets.copy_(o, non_blocking=True)
            if m is not None:
                ds.metadata.copy_(m, non_blocking=True)
            ds.validated = False
            ds.validate()                       # the reference decoder's checks, every call
            pipes[k].run(outs)                  # its statistics come back to the host (D2H) here
            moved += 80
            for out in (outs if copy_outputs else ()):   # every output element back to host memory
                flat = out.reshape(-1)
                for s in range(0, flat.numel(), stage.numel()):
                    n = min(stage.numel(), flat.numel() - s)
                    stage[:n].copy_(flat[s:s + n])
                    moved += 4 * n
        d2h = moved

    torch.cuda.synchronize()
    comm.barrier()
    t0 = time.perf_counter()
    for _ in range(args.e2e_steps):
        e2e_step()
    torch.cuda.synchronize()
    comm.barrier()
    dt = (time.perf_counter() - t0) / args.e2e_steps
    tt = torch.tensor([dt], dtype=torch.float64, device="cuda")
    comm.all_reduce(tt, "max")
    dt = float(tt.item())
    d2h_all = d2h
    # the same with the output fields left on the device (the API's out="torch" mode): only the
    # statistics come back; reported beside the headline, which copies every output to the host
    torch.cuda.synchronize()
    comm.barrier()
    t0 = time.perf_counter()
    for _ in range(args.e2e_steps):
        e2e_step(copy_outputs=False)
    torch.cuda.synchronize()
    comm.barrier()
    dtd = (time.perf_counter() - t0) / args.e2e_steps
    tt = torch.tensor([dtd], dtype=torch.float64, device="cuda")
    comm.all_reduce(tt, "max")
    dtd = float(tt.item())
    return {"value": round(len(KINDS) * 4.0 * n_total / dt / 1e9, 3), "unit": "GB/s",
            "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h_all), "s_per_step": round(dt, 3),
            "steps": args.e2e_steps, "path": "pinned host containers -> H2D -> hszg_validate -> windowed "
                                             "pipeline -> D2H of all four fp32 outputs (per rank)",
            "device_outputs": {"value": round(len(KINDS) * 4.0 * n_total / dtd / 1e9, 3), "unit": "GB/s",
                               "s_per_step": round(dtd, 3), "h2d_bytes_per_step": int(h2d),
                               "d2h_bytes_per_step": int(d2h),
                               "path": "same, outputs left on the device (statistics D2H only)"}}


def time_exact(args, pipes, outs, comm, step, n_total):
    """The headline step with the exact fp32 emitter (fp32 outputs = fl32 of the reference float64,
    bit-exact vs the oracle): W warm-up steps (graph re-capture), then K steps timed like the headline."""
    import torch

    for p in pipes.values():
        p.exact_fp32 = True
    for _ in range(max(2, args.warmup)):
        step()
    torch.cuda.synchronize()
    comm.barrier()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record()
    for _ in range(args.steps):
        step()
    ev1.record()
    torch.cuda.synchronize()
    comm.barrier()
    tt = torch.tensor([ev0.elapsed_time(ev1) / args.steps], dtype=torch.float64, device="cuda")
    comm.all_reduce(tt, "max")
    ms = float(tt.item())
    for p in pipes.values():
        p.exact_fp32 = False
    return {"ms_per_step": round(ms, 3), "value": round(len(KINDS) * 4.0 * n_total / (ms / 1e3) / 1e9, 2),
            "unit": "GB/s", "steps": args.steps}


def _plane_checksums(t, step=32):
    """Per-plane int64 sums of the fp32 bit patterns of one output (device, chunked)."""
    import torch

    return torch.cat([t[a:a + step].view(torch.int32).to(torch.int64).sum(dim=(1, 2))
                      for a in range(0, t.shape[0], step)])


def parity_probe(args, pipes, outs, comm, eps, dims, z0, z1):
    """Post-timed check of the timed configuration against the oracle (oracle/parity.py).

    Per rank, the first and last <= 9 planes of its slab (rank-boundary planes at N > 1; at N = 1 the
    top planes sit beyond flat index 2^32) in the fast emitter (<= 4*2^-24 relative) and the exact
    emitter (bit-exact): oracle = fields.py stencils on oracle.quantize of the regenerated field
    planes.  Rank 0 also decodes its first planes from the GPU containers with the oracle decoder and
    checks them against quantize.  Every plane of every output: per-plane checksums of HSZP_ND ==
    HSZX_ND (both derive from the same q), and the exact global sums equal across kinds and emitters.
    """
    import numpy as np
    import torch

    from oracle import hsz_oracle as O
    from oracle import parity as PAR
    from paper_2603_25206_b200 import synthetic

    t0 = time.time()
    N0 = dims[0]
    wins = [(z0, min(z1, z0 + 9)), (max(z0, z1 - 9), z1)]
    want = []
    qs = []
    for a, b in wins:
        s, e = max(0, a - 1), min(N0, b + 1)
        f = synthetic.gen_config5_slab(s, e, dims=dims).cpu().numpy()
        q = O.quantize(f, eps)
        za, zb, w = PAR.stencil_planes(q, s, N0, eps)
        want.append((a, b, [x[a - za:b - za] for x in w]))
        qs.append((s, q))
    container_ok = None
    if z0 == 0:
        # the oracle's own decode of the GPU containers' first planes (no carry needed at z0 = 0)
        container_ok = True
        s, q = qs[0]
        n1, n2 = dims[1], dims[2]
        for k, p in pipes.items():
            ds = p.ds
            nplanes = 8 if k == 3 else min(10, q.shape[0])
            if k == 1:
                c1 = nplanes * (ds.n_chunks // p.sf.nz)
                m1 = 0
            else:
                from paper_2603_25206_b200.device import _full_row_chunks

                c1 = _full_row_chunks(ds)
                m1 = (n1 // 8) * (n2 // 8)
            c1 = min(c1, ds.n_chunks)
            hi = int(ds.offsets[c1].item()) if c1 < ds.n_chunks else ds.payload_len
            offs = ds.offsets[:c1].cpu().numpy().view(np.uint64)
            payload = ds.payload[:hi].cpu().numpy().tobytes()
            meta = None if ds.metadata is None else ds.metadata[:m1].cpu().numpy()
            st = PAR.sub_stream(k, dims, (8, 8, 8), eps, payload, offs, meta, 0, c1, 0, m1, nplanes=nplanes)
            container_ok &= bool(np.array_equal(O.stage3(st), q[:nplanes]))
    rec = {"exact": {}, "fast": {}}
    sums = {}
    for mode in ("fast", "exact"):
        for k, p in pipes.items():
            p.exact_fp32 = mode == "exact"
            res = p.run(outs)
            sums[(mode, k)] = (res["s1"], res["s2"])
            worst, ok, n = 0.0, True, 0
            for a, b, w in want:
                r = PAR.compare([o[a - z0:b - z0].cpu().numpy() for o in outs], w, mode == "exact")
                worst, ok, n = max(worst, r["max_rel_err"]), ok and r["ok"], n + r["values"]
            rec[mode][k] = {"ok": ok, "max_rel_err": worst, "values": n,
                            "checksums": torch.stack([_plane_checksums(o) for o in outs])}
        p.exact_fp32 = False
    for p in pipes.values():
        p.exact_fp32 = False
    same_ck = all(torch.equal(rec[m][1]["checksums"], rec[m][3]["checksums"]) for m in rec)
    same_sums = len(set(sums.values())) == 1
    flags = torch.tensor([float(all(rec["exact"][k]["ok"] for k in pipes)),
                          float(all(rec["fast"][k]["ok"] for k in pipes)), float(same_ck), float(same_sums),
                          float(container_ok if container_ok is not None else 1.0)], dtype=torch.float64,
                         device="cuda")
    comm.all_reduce(flags, "min")
    worst = torch.tensor([max(rec["fast"][k]["max_rel_err"] for k in pipes),
                          max(rec["exact"][k]["max_rel_err"] for k in pipes)], dtype=torch.float64, device="cuda")
    comm.all_reduce(worst, "max")
    nval = torch.tensor([float(sum(rec["fast"][k]["values"] for k in pipes))], dtype=torch.float64, device="cuda")
    comm.all_reduce(nval, "sum")
    f = [bool(x) for x in flags.cpu().tolist()]
    w = worst.cpu().tolist()
    return {"planes_rank0": [list(x) for x in wins], "values_checked_per_mode": int(nval.item()),
            "exact_bit_exact": f[0], "fast_within_tol": f[1], "fast_tol_rel": PAR.FAST_RTOL,
            "fast_max_rel_err": w[0], "exact_max_rel_err_vs_f64": w[1],
            "all_planes_hszp_nd_eq_hszx_nd": f[2], "bit_exact_sums_across_kinds_and_emitters": f[3],
            "rank0_container_decode_eq_quantize": f[4],
            "oracle": "oracle/parity.py: fields.py:34-80 stencils on quantize (quant.py:69-82) of the regenerated "
                      "field planes; oracle decoder on the GPU containers (rank 0)",
            "seconds": round(time.time() - t0, 1)}


CPU_SECONDS = 10.0


def measured_traffic(op, dims, world, window):
    """DRAM bytes per step of an op from the committed ncu `--set full` captures of its kernels
    (profiles/r02_traffic.json; r01_traffic.json as a fallback), when they were taken on this exact shape (config 5, 1 GPU, W = 64)."""
    prof = os.path.join(os.path.dirname(os.path.abspath(__file__)), "profiles")
    name = "r02_traffic.json" if os.path.exists(os.path.join(prof, "r02_traffic.json")) else "r01_traffic.json"
    path = os.path.join(prof, name)
    try:
        with open(path) as f:
            rec = json.load(f)["ops"].get(op)
    except (OSError, ValueError, KeyError):
        return None
    if rec is None or tuple(dims) != (2048, 2048, 2048) or world != 1 or window != 64:
        return None
    return {"traffic_bytes_per_step": int(rec["traffic_bytes_per_step"]),
            "source": f"profiles/{name}: ncu --set full of " + ", ".join(rec["kernels"])}


def build_cpu_sample(field_dev, eps):
    """The CPU sample's containers, compressed on the GPU (bit-identical to oracle.compress)."""
    from oracle import cpu_pipeline as CP
    from oracle import hsz_oracle as O
    from paper_2603_25206_b200.compressors import compress_device

    S = CP.sample_planes(CP.host_cores())
    blobs = []
    Z, N1, N2 = field_dev.shape
    for z in range(0, min(S, Z) - CP.SUB_PLANES + 1, CP.SUB_PLANES):
        for y in range(0, N1 - CP.SUB_ROWS + 1, CP.SUB_ROWS):
            sub = field_dev[z:z + CP.SUB_PLANES, y:y + CP.SUB_ROWS].contiguous()
            for kind in KINDS:
                ds = compress_device(sub, kind, eps, (8, 8, 8))
                meta = None if ds.metadata is None else ds.metadata.cpu().numpy().copy()
                st = O.Stream(kind, ds.dims, ds.block_dims, eps, meta, ds.offsets.cpu().numpy().view("u8").copy(),
                              ds.payload[:ds.payload_len].cpu().numpy().tobytes())
                blobs.append(O.stream_to_bytes(st))
    return blobs


def cpu_measure(blobs, seconds: float, steps: int | None = None, warmup: int = 1):
    """The reference CPU path on the sample: every container decoded by the reference's Cython codec
    (oracle/_ref, _bitpack.pyx) then recorrelated / summed / differenced with the reference's numpy
    expressions (oracle restatement), one container per worker process.

    all-core: a step = one pass over the sample on a pool of one process per host core (`steps` timed
    passes after `warmup`, or as many as fill `seconds`); one-thread: containers run in this process
    one after another for about a third of `seconds` (the reference is single-threaded by contract,
    SPEC.md:286)."""
    from oracle import cpu_pipeline as CP

    cores = CP.host_cores()
    pool = CP.make_pool(cores)
    for _ in range(max(1, warmup)):
        CP.run_sample(blobs, pool)
    times, elems = [], 0
    while (steps is not None and len(times) < steps) or (steps is None and (not times or sum(times) < seconds)):
        dt, elems, _ = CP.run_sample(blobs, pool)
        times.append(dt)
    if pool is not None:
        pool.shutdown()
    dt = sum(times) / len(times)
    t0 = time.perf_counter()
    n1, e1 = 0, 0
    while n1 < len(blobs) and (n1 < 2 or time.perf_counter() - t0 < seconds / 3):
        _, e, _ = CP.run_sample([blobs[n1]], None)
        e1 += e
        n1 += 1
    d1 = time.perf_counter() - t0
    codec = "reference Cython _bitpack (oracle/_ref)" if CP.ref_codec() else "oracle C codec (oracle/_ref not built)"
    return {"value": round(4.0 * elems / dt / 1e9, 4), "unit": "GB/s", "cores": cores,
            "kind": "reference" if CP.ref_codec() else "port", "ms_per_pass": round(dt * 1e3, 1),
            "passes": len(times),
            "one_thread": {"value": round(4.0 * e1 / d1 / 1e9, 4), "unit": "GB/s", "cores": 1, "containers": n1},
            "sample": f"{len(blobs)} containers of {CP.SUB_PLANES}x{CP.SUB_ROWS}x2048 sub-fields of planes "
                      f"[0, {CP.sample_planes(cores)}) of the config-5 field (HSZP_ND + HSZX_ND, global eps), "
                      f"{elems} values per pass; per container: decode ({codec}) + recorrelate + exact sum/sumsq "
                      f"+ 3-comp gradient + Laplacian (reference numpy expressions); {min(cores, len(blobs))} "
                      f"processes", "same_config": True}


def cpu_baseline(blobs, seconds=CPU_SECONDS):
    return cpu_measure(blobs, seconds)


# ---------------------------------------------------------------------------
# reference arm


def reference_containers(dims):
    """The CPU sample's containers exactly as the GPU arm builds them: config-5 field generated on the
    device, eps = 1e-3 x the GLOBAL value range (min/max over every plane), sub-fields compressed
    (bit-identical to oracle.compress, tests/test_gpu_api.py)."""
    import torch

    from oracle import cpu_pipeline as CP
    from paper_2603_25206_b200 import synthetic
    from paper_2603_25206_b200.quant import field_minmax

    N0 = dims[0]
    lo, hi = math.inf, -math.inf
    for z in range(0, N0, 128):
        f = synthetic.gen_config5_slab(z, min(N0, z + 128), dims=dims)
        a, b, _ = field_minmax(f.reshape(-1))
        lo, hi = min(lo, a), max(hi, b)
        del f
    eps = 1e-3 * (hi - lo)
    S = CP.sample_planes(CP.host_cores())
    f = synthetic.gen_config5_slab(0, S, dims=dims)
    blobs = build_cpu_sample(f, eps)
    del f
    torch.cuda.empty_cache()
    return blobs, eps


def run_reference(args):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    import torch

    torch.cuda.set_device(0)
    N0, N1, N2 = args.dims
    t0 = time.time()
    blobs, eps = reference_containers((N0, N1, N2))
    setup_s = time.time() - t0
    cpu = cpu_measure(blobs, CPU_SECONDS, steps=args.steps, warmup=args.warmup)
    value = cpu["value"]
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": "GB/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": cpu["ms_per_pass"], "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "int32",
            "data": "synthetic: config-5 field (device generator, seed 5), the GPU arm's CPU-sample containers",
            "config": {"workload": "config5 bounded sample: per sub-field container decode (reference Cython codec) "
                                   "+ recorrelate + exact mean/variance sums + 3-comp gradient + Laplacian",
                       "dims": [N0, N1, N2], "kinds": [KIND_NAMES[k] for k in KINDS], "eps": eps,
                       "setup_s": round(setup_s, 1)},
            "cpu_baseline": cpu,
            "e2e": {"value": value, "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def spawn(args):
    """--gpus N without a torchrun environment: re-launch this command as N ranks (one per GPU)."""
    import socket

    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", str(args.gpus),
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
    env = dict(os.environ)
    env.setdefault("NCCL_DEBUG", "INFO")
    env.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    return subprocess.call(cmd, env=env)


def main():
    args = parse()
    if args.impl == "ours" and args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(spawn(args))
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
