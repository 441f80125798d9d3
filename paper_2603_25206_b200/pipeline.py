"""Windowed, z-slab-sharded analytics over 3-D compressed fields.

Two reference mechanisms meet here:

* Algorithm 3, the out-of-core sliding window (stages.py:173-258,
  fields.py:243-272): a rank walks its planes in windows of
  W planes, reconstructing q into a small device buffer (prefix carry for
  HSZP_ND, block-row granularity for HSZX_ND) and running the fused
  gradient+Laplacian stencil on it, so q is never materialised for the whole
  field (2048^3 outputs alone are 137 GB of HBM).
* the z-slab partition of SURVEY §8(e) across 1/2/4/8 GPUs (one process per
  GPU, torch.distributed over NCCL): every rank owns planes [z0, z1) of the
  global stream (a contiguous chunk range, bit-identical to the global
  container), exchanges one int32 halo plane with each neighbour, HSZP_ND
  ranks combine their slab-total planes with one all-gather (Lorenzo carry,
  exact in int32 wrap-around), and the global mean/variance is the exact
  int128 combination of the per-rank sums (one all-gather of 64-byte
  records; Python-int finalisation as stats.py:58-62).

The exchange helpers only use torch.distributed collectives on tensors, so
the same code runs on NCCL/CUDA in production and on gloo/CPU in the
multi-process CPU tests.
"""

from __future__ import annotations

import ctypes
import math
from dataclasses import dataclass

import numpy as np

from . import _lib
from ._nvtx import ranged

_SMS = 148          # B200 SM count (grid sizing only)
FUSED_LAYERS = 16   # block layers (8 planes each) per CTA of the one-pass kernels
FAST_QLIM = 1 << 27  # fast fp32 emitter validity bound on |q| (stencil.cuh)
EM_FAST, EM_EXACT, EM_TABLE = 0, 1, 2   # emitter modes of the fused kernels (stencil.cuh EmitMode)

HSZP_ND, HSZX_ND = 1, 3
SUMS_BYTES = 64

# The configuration bench.py times (and tests/test_gpu_headline.py checks against the oracle): CUDA-graph
# replay of the window loop, HSZX_ND one-pass kernel, HSZP_ND persistent side-stream band scans (band height
# sized by _band_rows: 256 rows at 2048^2 planes) under the ring z-sweeps, fast fp32 emitter.
HEADLINE_SETTINGS = dict(use_graph=True, exact_fp32=False, one_pass=True, lorenzo_one_pass=False, overlap=True,
                         band_rows_req=None)
SETTINGS = ("use_graph", "exact_fp32", "exact_table", "one_pass", "lorenzo_one_pass", "overlap", "band_rows_req", "fused_layers")


def apply_settings(pipe, **kw):
    """Set pipeline options by name (unknown names are an error); cached buffers and the captured
    graph are rebuilt on the next run when a setting they depend on changed (_settings_key)."""
    for k, v in kw.items():
        if k not in SETTINGS:
            raise ValueError(f"unknown pipeline setting {k!r}")
        setattr(pipe, k, v)
    return pipe


# ---------------------------------------------------------------------------
# communication plumbing


class Comm:
    """Rank/world and the few collectives the pipeline needs (no-ops at world size 1)."""

    @classmethod
    def local(cls):
        """A world-1 communicator regardless of any initialised process group (single-GPU API calls)."""
        c = cls.__new__(cls)
        c.dist, c.group, c.rank, c.world, c.host_staged = None, None, 0, 1, False
        return c

    def __init__(self, group=None):
        try:
            import torch.distributed as dist

            ok = dist.is_available() and dist.is_initialized()
        except Exception:  # noqa: BLE001
            ok = False
        self.dist = dist if ok else None
        self.group = group
        self.rank = dist.get_rank(group) if ok else 0
        self.world = dist.get_world_size(group) if ok else 1
        # gloo moves host tensors: device tensors are staged through host copies (CPU tests, and
        # plumbing checks with several ranks on one GPU); NCCL takes device tensors directly
        self.host_staged = ok and dist.get_backend(group) == "gloo"

    def _host(self, t):
        return t.cpu() if (self.host_staged and t.is_cuda) else t

    def all_gather(self, t):
        """List of every rank's tensor (same shape/dtype)."""
        if self.world == 1:
            return [t]
        import torch

        h = self._host(t.contiguous())
        outs = [torch.empty_like(h) for _ in range(self.world)]
        self.dist.all_gather(outs, h, group=self.group)
        return [o.to(t.device) for o in outs] if h is not t else outs

    def all_reduce(self, t, op: str):
        if self.world == 1:
            return t
        ops = {"sum": self.dist.ReduceOp.SUM, "min": self.dist.ReduceOp.MIN, "max": self.dist.ReduceOp.MAX}
        h = self._host(t)
        self.dist.all_reduce(h, op=ops[op], group=self.group)
        if h is not t:
            t.copy_(h)
        return t

    def exchange(self, to_lower, to_upper, like):
        """Send `to_lower` to rank-1 and `to_upper` to rank+1; return (from_lower, from_upper).

        `like` gives the shape/dtype/device of the received planes; missing neighbours give None.
        """
        if self.world == 1:
            return None, None
        import torch

        ops = []
        from_lower = from_upper = None
        r, w = self.rank, self.world
        like_h = self._host(like)
        P2P = self.dist.P2POp
        if r > 0:
            from_lower = torch.empty_like(like_h)
            ops.append(P2P(self.dist.irecv, from_lower, r - 1, group=self.group))
            ops.append(P2P(self.dist.isend, self._host(to_lower.contiguous()), r - 1, group=self.group))
        if r < w - 1:
            from_upper = torch.empty_like(like_h)
            ops.append(P2P(self.dist.irecv, from_upper, r + 1, group=self.group))
            ops.append(P2P(self.dist.isend, self._host(to_upper.contiguous()), r + 1, group=self.group))
        # one grouped launch (ncclGroupStart/End under NCCL): separately issued send/recv pairs
        # whose both ends start with a recv would wait on each other
        for q in self.dist.batch_isend_irecv(ops) if ops else []:
            q.wait()
        if like_h is not like:
            from_lower = None if from_lower is None else from_lower.to(like.device)
            from_upper = None if from_upper is None else from_upper.to(like.device)
        return from_lower, from_upper

    def barrier(self):
        if self.world > 1:
            self.dist.barrier(group=self.group)


def shard_planes(n0: int, world: int, rank: int, align: int = 16) -> tuple:
    """Rank's plane range [z0, z1): contiguous, boundaries multiples of `align` (block depth x region)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank/world")
    units = -(-n0 // align)
    bounds = [min(n0, (units * r // world) * align) for r in range(world + 1)]
    bounds[-1] = n0
    z0, z1 = bounds[rank], bounds[rank + 1]
    if z1 <= z0:
        raise ValueError(f"{n0} planes cannot feed {world} ranks at {align}-plane alignment")
    return z0, z1


def exclusive_plane_prefix(planes, rank: int):
    """C_rank = sum_{g < rank} T_g (int32 wrap-around) — the Lorenzo carry of a z-slab."""
    import torch

    acc = torch.zeros_like(planes[0])
    if acc.is_cuda:                          # one wrap-around int32 add kernel per lower rank (hszg_add_plane)
        for g in range(rank):
            src = planes[g].contiguous()
            _lib.call("hszg_add_plane", _lib.ptr(acc), _lib.ptr(src), acc.numel(), acc.numel(), _lib.stream_handle())
        return acc
    for g in range(rank):                    # host tensors (gloo CPU tests): the same arithmetic in int64
        acc = (acc.to(torch.int64) + planes[g].to(torch.int64)).remainder(2**32)
        acc = torch.where(acc >= 2**31, acc - 2**32, acc).to(planes[0].dtype)
    return acc


def sums_to_ints(buf) -> dict:
    """Decode one 64-byte HszgSums record (host bytes or tensor) into exact Python ints."""
    raw = bytes(buf.cpu().numpy().tobytes()) if hasattr(buf, "cpu") else bytes(buf)
    s = _lib.Sums.from_buffer_copy(raw)
    return dict(s1=s.s1, s2=s.s2, count=int(s.count), vmin=int(s.vmin), vmax=int(s.vmax))


ACC_BYTES = 80     # sizeof(HszgAcc)


def acc_to_ints(buf) -> dict:
    """Decode an HszgAcc (32-bit limbs of the int128 sums, limb 3 signed) into exact Python ints."""
    raw = bytes(buf.cpu().numpy().tobytes()) if hasattr(buf, "cpu") else bytes(buf)
    u = np.frombuffer(raw[:72], dtype="<u8").astype(object)
    cnt = int(np.frombuffer(raw[64:72], dtype="<i8")[0])
    vmin, vmax = (int(v) for v in np.frombuffer(raw[72:80], dtype="<i4"))

    def val(limbs):
        top = int(limbs[3])
        top = top - 2**64 if top >= 2**63 else top
        return int(limbs[0]) + (int(limbs[1]) << 32) + (int(limbs[2]) << 64) + (top << 96)

    return dict(s1=val(u[0:4]), s2=val(u[4:8]), count=cnt, vmin=vmin, vmax=vmax)


def combine_rank_sums(comm: Comm, local_sums_buf) -> dict:
    """Exact global (sum q, sum q^2, count, min, max) from every rank's int128 record (one all-gather)."""
    parts = comm.all_gather(local_sums_buf)
    tot = dict(s1=0, s2=0, count=0, vmin=2**31, vmax=-(2**31))
    for p in parts:
        d = sums_to_ints(p)
        tot["s1"] += d["s1"]
        tot["s2"] += d["s2"]
        tot["count"] += d["count"]
        tot["vmin"] = min(tot["vmin"], d["vmin"])
        tot["vmax"] = max(tot["vmax"], d["vmax"])
    return tot


def finalize_mean_var(s1: int, s2: int, n: int, eps: float) -> tuple:
    """(mean, variance) with the reference's exact expressions (stats.py:58-62, 115-118; N1)."""
    mean = s1 / n * (2.0 * eps)
    var = (s2 * n - s1 * s1) / (n * (n - 1)) * ((2.0 * eps) * (2.0 * eps))
    return mean, var


# ---------------------------------------------------------------------------
# sharded containers


@dataclass
class ShardedField:
    """One rank's share of a z-partitioned 3-D compressed field."""

    kind: int
    eps: float
    global_dims: tuple      # (N0, n1, n2)
    block_dims: tuple
    z0: int
    z1: int
    ds: object              # DeviceStream over planes [z0, z1)

    @property
    def nz(self) -> int:
        return self.z1 - self.z0


def compress_shard(field_dev, kind: int, eps: float, block_dims, z0: int, z1: int, global_dims) -> ShardedField:
    """Compress planes [z0, z1) so the chunks equal the global stream's chunk range for those planes.

    field_dev holds planes [z0 - lead, z1) where lead = 1 for HSZP_ND with z0 > 0 (the Lorenzo
    predictor reads the previous plane; the lead plane's chunks are dropped — SURVEY §8(c)), else 0.
    HSZX_ND needs z0 on a block-row boundary.  eps must be the GLOBAL absolute bound.
    """
    from .compressors import compress_device
    from .device import DeviceStream

    t = _lib.torch()
    lead = 1 if (kind == HSZP_ND and z0 > 0) else 0
    if field_dev.shape[0] != z1 - z0 + lead:
        raise ValueError("field slab does not match the plane range (+ lead plane)")
    if kind == HSZX_ND and z0 % block_dims[0]:
        raise ValueError("HSZX_ND shards must start on a block-row boundary")
    dims = tuple(field_dev.shape)
    bd = tuple(min(b, n) for b, n in zip(block_dims, dims))
    full = compress_device(field_dev, kind, eps, bd)
    if not lead:
        return ShardedField(kind, eps, tuple(global_dims), tuple(block_dims), z0, z1, full)
    cpp = full.n_chunks // dims[0]
    off0 = int(full.offsets[cpp].item())
    plen = full.payload_len - off0
    payload = t.zeros(plen + _lib.PAYLOAD_PAD, dtype=t.uint8, device=_lib.device())
    payload[:plen].copy_(full.payload[off0:full.payload_len])
    offs = full.offsets[cpp:] - off0
    local_dims = (z1 - z0,) + dims[1:]
    local_bd = tuple(min(b, n) for b, n in zip(block_dims, local_dims))
    ds = DeviceStream(kind, local_dims, local_bd, eps, payload, plen, offs.contiguous(), None)
    del full
    return ShardedField(kind, eps, tuple(global_dims), tuple(block_dims), z0, z1, ds)


# ---------------------------------------------------------------------------
# the windowed pipeline


class WindowPipeline:
    """Global mean/variance + 3-component gradient + Laplacian of one rank's shard, window by window."""

    def __init__(self, sf: ShardedField, comm: Comm | None = None, window: int = 64):
        t = _lib.torch()
        self.sf = sf
        self.comm = comm or Comm()
        self.ds = sf.ds.validate()
        self.G = 1 if sf.kind == HSZP_ND else sf.ds.block_dims[0]
        self.W = max(self.G, (window // self.G) * self.G)
        n1, n2 = sf.global_dims[1], sf.global_dims[2]
        self.plane = n1 * n2
        self._buf = None            # general-loop window buffer, allocated on first use
        self.nwin = -(-sf.nz // self.W)
        self.win_sums = t.zeros(max(self.nwin, 1) * SUMS_BYTES, dtype=t.uint8, device=_lib.device())
        self.halo_lo = None
        self.halo_hi = None
        self.timer = None          # optional EventTimer (bench.py): CUDA events per launch group

    def _range_bytes(self, s: int, e: int) -> int:
        """Compressed bytes of local planes [s, e): payload range + 8 B per chunk + 4 B per block mean."""
        if not hasattr(self, "_plane_off"):
            # byte offset / chunk index of every window-aligned plane boundary, fetched once (small D2H)
            t = _lib.torch()
            nz, nc = self.sf.nz, self.ds.n_chunks
            if self.sf.kind == HSZP_ND:
                per = nc // nz
                chunks = [z * per for z in range(nz)]
            else:
                from .device import _full_row_chunks

                rc = _full_row_chunks(self.ds)
                chunks = [(z // self.G) * rc for z in range(nz)]
            idx = t.tensor([min(c, nc - 1) for c in chunks], dtype=t.int64, device=self.ds.offsets.device)
            offs = self.ds.offsets.index_select(0, idx).cpu().numpy().tolist()
            self._plane_chunk = chunks + [nc]
            self._plane_off = [o if c < nc else self.ds.payload_len for o, c in zip(offs, chunks)] + [
                self.ds.payload_len]
        c0, c1 = self._plane_chunk[s], self._plane_chunk[e]
        p0, p1 = self._plane_off[s], self._plane_off[e]
        meta = 0 if self.ds.metadata is None else 4 * self.ds.metadata.numel() * (e - s) // self.sf.nz
        return (p1 - p0) + 8 * (c1 - c0) + meta

    # -- per-container collective setup (inside the timed step: it depends on the data) -------
    def _decode_planes(self, s: int, e: int, out):
        """q of local planes [s, e) into `out` (no carry)."""
        sub = self.ds.plane_view(s, e)
        return sub.reconstruct(_lib.torch().int32, out=out)

    def prepare(self):
        comm = self.comm
        self._agree_paths()
        if comm.world == 1:
            # no neighbours: no halo planes, no Lorenzo carry (z0 = 0) — nothing to decode here
            self.apply_boundary(None, None, None)
            return
        ct = self.comm_timer
        if ct:
            ct.begin("boundary_decode")
        mine = self.local_boundary(need_total=True)
        if ct:
            ct.end("boundary_decode", 0)
            ct.begin("carry_allgather")
        gathered = comm.all_gather(mine["T"]) if mine.get("T") is not None else None
        carry = self.carry_from(gathered, comm.rank)
        first = self.finish_first(mine, carry)
        if ct:
            ct.end("carry_allgather", 0)
            ct.begin("halo_exchange")
        lo, hi = comm.exchange(first if first is not None else mine["head"], mine["tail"], mine["tail"])
        if ct:
            ct.end("halo_exchange", 0)
        self.apply_boundary(carry, lo, hi)

    comm_timer = None   # optional EventTimer (bench.py): the boundary / collective phases outside the graph

    def _agree_paths(self):
        """Every rank must take the same kernel path (the paths issue different collectives): the
        data-dependent eligibility flags (canonical index, bit widths <= 16) are agreed with one MIN
        all-reduce, once per container."""
        if getattr(self, "_agreed", None) is not None:
            return
        t = _lib.torch()
        flags = t.tensor([int(bool(self.ds.desc.canonical)), int(self.ds.desc.max_bitwidth <= 16)],
                         dtype=t.int32, device=_lib.device())
        self.comm.all_reduce(flags, "min")
        self._agreed = tuple(bool(v) for v in flags.cpu().tolist())

    def _canonical(self) -> bool:
        a = getattr(self, "_agreed", None)
        return a[0] if a is not None else bool(self.ds.desc.canonical)

    def _narrow_bw(self) -> bool:
        a = getattr(self, "_agreed", None)
        return a[1] if a is not None else self.ds.desc.max_bitwidth <= 16

    # The three phases below are split so a multi-rank run can also be emulated rank by rank
    # in one process (tests/test_gpu_pipeline.py); prepare() runs them around the collectives.
    def local_boundary(self, need_total: bool) -> dict:
        """Boundary planes computable from this rank's bytes alone.

        HSZP_ND: the local 2-D prefix of the first plane, and (multi-rank) the slab total
        T = P2(sum_z p) whose exclusive prefix over ranks is the Lorenzo carry.
        HSZX_ND: q of the first and last planes (halos of the neighbours).
        """
        t = _lib.torch()
        sf = self.sf
        n1, n2 = sf.global_dims[1], sf.global_dims[2]
        out = {"T": None, "head": None, "tail": None}
        if sf.kind == HSZP_ND:
            first = t.empty((1, n1, n2), dtype=t.int32, device=_lib.device())
            self._decode_planes(0, 1, first)                     # P2(p[z0]) (local prefix)
            out["first_local"] = first
            if need_total:
                U = t.empty((n1, n2), dtype=t.int32, device=_lib.device())
                err = _lib.Err()
                _lib.call("hszg_plane_sum", ctypes.byref(self.ds.geom), ctypes.byref(self.ds.desc), _lib.ptr(U),
                          _lib.stream_handle(), ctypes.byref(err), err=err)
                out["T"] = _plane_prefix(U)                      # slab total = P2(sum_z p)
            out["tail"] = first[0]                               # placeholder shape for the exchange
        else:
            B0 = self.G
            lo_rows = min(B0, sf.nz)
            head = t.empty((lo_rows, n1, n2), dtype=t.int32, device=_lib.device())
            self._decode_planes(0, lo_rows, head)
            s_last = ((sf.nz - 1) // B0) * B0
            tail = t.empty((sf.nz - s_last, n1, n2), dtype=t.int32, device=_lib.device())
            self._decode_planes(s_last, sf.nz, tail)
            out["head"], out["tail"] = head[0], tail[-1]
        return out

    def carry_from(self, gathered_T, rank: int):
        """HSZP_ND carry C_rank = q[z0 - 1] from every rank's slab total (None for HSZX_ND)."""
        if self.sf.kind != HSZP_ND:
            return None
        t = _lib.torch()
        n1, n2 = self.sf.global_dims[1], self.sf.global_dims[2]
        if gathered_T is None:
            return t.zeros((n1, n2), dtype=t.int32, device=_lib.device())
        return exclusive_plane_prefix(gathered_T, rank)

    def finish_first(self, mine: dict, carry):
        """HSZP_ND: q[z0] = C + P2(p[z0]) — the plane sent to rank-1 as its upper halo."""
        if self.sf.kind != HSZP_ND:
            return None
        first = mine["first_local"]
        _lib.call("hszg_add_plane", _lib.ptr(first), _lib.ptr(carry), self.plane, self.plane, _lib.stream_handle())
        return first[0]

    def apply_boundary(self, carry, from_lower, from_upper):
        self.carry = carry                                       # = q[z0 - 1] (HSZP_ND)
        if self.sf.kind == HSZP_ND:
            self.halo_lo = carry if self.sf.z0 > 0 else None
        else:
            self.halo_lo = from_lower
        self.halo_hi = from_upper

    def run_prepared(self, outs, stats: bool = True):
        """run() after the boundary phases were applied by the caller (single-process emulation)."""
        return self.run(outs, stats, _prepared=True)

    # -- the windowed pass ---------------------------------------------------------------
    def _check_outs(self, outs):
        """outs must be four distinct contiguous float32 / float64 CUDA tensors of the slab's shape (the
        kernels write every output; a null or short output would be written out of bounds)."""
        t = _lib.torch()
        shape = (self.sf.nz,) + tuple(self.sf.global_dims[1:])
        if len(outs) != 4 or any(o is None for o in outs):
            raise ValueError("WindowPipeline.run needs four output tensors [dz, dy, dx, laplacian]")
        for o in outs:
            if (tuple(o.shape) != shape or o.dtype not in (t.float32, t.float64) or not o.is_cuda
                    or not o.is_contiguous()):
                raise ValueError(f"pipeline outputs must be contiguous float CUDA tensors of shape {shape}")
        if len({o.data_ptr() for o in outs}) != 4:
            raise ValueError("pipeline outputs must not alias")

    def _fast_ok(self, outs) -> bool:
        """The fused window kernels need rows of whole chunks (HSZP_ND), 16-B rows and fp32 outputs."""
        t = _lib.torch()
        n2 = self.sf.global_dims[2]
        o = outs[0]
        if n2 % 4 or o.dtype != t.float32 or not self._canonical():
            return False
        if self.sf.kind == HSZP_ND:
            return n2 % 32 == 0 and n2 <= 4096
        return True

    @ranged("hsz/pipeline_run")
    def run(self, outs, stats: bool = True, _prepared: bool = False):
        """Fill outs = [dz, dy, dx, laplacian] (float tensors of shape (nz, n1, n2)); return global stats.

        With ``use_graph`` the whole window loop (hundreds of launches) is captured once into a CUDA
        graph and replayed; the per-container boundary phase (halos / carry, collectives) and the
        final stats read-back stay outside it.
        """
        self._check_outs(outs)
        if not _prepared:
            self.prepare()
        if self._fast_ok(outs):
            self._stage_boundary()
            if self.use_graph:
                self._replay(outs)
            else:
                self._fused_loop(outs)
            res = self._finish_stats(_prepared) if stats else None
            ovf = self._l_overflow(_prepared)
            if ovf:
                # a narrow band-local prefix did not fit: widen (int8 -> int16, int16 -> int32; kept from
                # now on) and redo the pass
                if ovf & 2:
                    self.l16 = False
                self.l8 = False
                self._pers_W = None
                self._stage_boundary()
                self._fused_loop(outs)
                res = self._finish_stats(_prepared) if stats else None
                if self._l_overflow(_prepared):
                    self.l16 = False
                    self._pers_W = None
                    self._stage_boundary()
                    self._fused_loop(outs)
                    res = self._finish_stats(_prepared) if stats else None
            if self._emit_mode() != EM_EXACT and not self._fast_valid(
                    res if stats else self._finish_stats(_prepared), _prepared):
                # the fast and table emitters compute the stencils in int32, valid while |q| < 2^27
                # (FAST_QLIM, stencil.cuh): every q is some point's centre, so the exact min / max decide
                # it; redo the pass with the fp64-conversion exact emitter
                self._force_exact64 = True
                try:
                    self._fused_loop(outs)
                    res = self._finish_stats(_prepared)
                finally:
                    self._force_exact64 = False
            return res if stats else None
        return self._run_generic(outs, stats, _prepared)

    # HSZP_ND two-pass: band-local prefixes L stored narrow — int8 (a quarter of the int32 traffic)
    # except in the window holding the field's first plane (there L is the y-difference of q itself,
    # int16), or int16 everywhere; a device flag (bit 1: int8, bit 2: int16) reports any value that did
    # not fit and the pass is redone one width up
    l16 = True
    l8 = True

    def _l16_active(self) -> bool:
        # narrow L feeds only the ring z-sweep (band rows a multiple of 16)
        return bool(self.band_rows) and self.band_rows % 16 == 0 and self.l16 and self.sf.global_dims[2] % 8 == 0

    def _l_mode(self, a: int) -> int:
        """Width code of window [a, ...)'s L: 0 int32, 1 int16, 2 int8."""
        if not self._l16_active():
            return 0
        if self.l8 and self.sf.global_dims[2] % 16 == 0 and self.sf.z0 + a > 0:
            return 2
        return 1

    def _l_overflow(self, _prepared) -> int:
        if not getattr(self, "_l16_used", False):
            return 0
        flag = self.l16_ovf.clone()
        if not _prepared:
            self.comm.all_reduce(flag, "max")          # every rank redoes the pass together
        return int(flag.item())

    def _l16_overflowed(self, _prepared) -> bool:
        return self._l_overflow(_prepared) != 0

    def _fast_valid(self, res, _prepared) -> bool:
        lim = FAST_QLIM
        ok = -lim < res["vmin"] and res["vmax"] < lim
        if _prepared:       # local stats only: the neighbours' halo planes are checked here
            for h in (self.halo_lo, self.halo_hi):
                if h is not None and int(h.abs().max()) >= lim:
                    ok = False
        return ok

    use_graph = False
    # fp32 outputs of the fused loop: True = fl32 of the reference float64 (bit-exact vs the oracle);
    # False = int32 stencil x fl32(eps) in fp32 (<= 2^-23 relative, no fp64 conversions: faster).
    exact_fp32 = False
    # exact mode by table (EM_TABLE, stencil.cuh): bit-identical to the fp64-conversion emitter; off = always
    # the conversion chain (tests compare the two)
    exact_table = True
    _force_exact64 = False

    def _emit_mode(self) -> int:
        """Emitter mode of the fused kernels: EM_FAST, EM_EXACT (fp64 conversions) or EM_TABLE."""
        if self._force_exact64:
            return EM_EXACT
        if not self.exact_fp32:
            return EM_FAST
        eps = float(self.sf.eps)
        return EM_TABLE if (self.exact_table and 2.0 ** -125 <= eps <= 2.0 ** 90) else EM_EXACT
    band_rows_req = None        # force a band height for hszg_band_scan (tests); None: sized for the grid

    # -- fused loops (window.cu) ---------------------------------------------------------------
    def _persistent(self):
        """Buffers whose addresses stay fixed across runs (graph-capture safe)."""
        t = _lib.torch()
        key = (self.W, self.band_rows_req, self.one_pass, self.lorenzo_one_pass, self.l16, self.l8, self.overlap)
        if getattr(self, "_pers_W", None) == self.W and getattr(self, "_pers_key", None) == key:
            return
        n1, n2 = self.sf.global_dims[1], self.sf.global_dims[2]
        dev = _lib.device()
        one = self._one_pass_ok()
        nslots = 0 if one else 3
        self.band_rows = self._band_rows() if (self.sf.kind == HSZP_ND and not one) else 0
        rtype = t.int16 if self._l16_active() else t.int32
        self.ring = [t.empty((self.W, n1, n2), dtype=rtype, device=dev) for _ in range(nslots)]
        if one and self.sf.kind == HSZP_ND:
            nz = self.sf.nz
            self.lz_bands = t.empty((nz, -(-n1 // 16), n2), dtype=t.int32, device=dev)
            self.lz_edges = t.empty(nz * -(-n2 // 128) * ((n1 + 1) // 2 * 2) * 2 + 64, dtype=t.int32, device=dev)
        self.halo_buf = t.zeros((2, n1, n2), dtype=t.int32, device=dev)       # [lower, upper]
        self.carry_buf = t.zeros((3, n1, n2), dtype=t.int32, device=dev)      # [rank carry, ping, pong]
        self.acc = t.zeros(ACC_BYTES, dtype=t.uint8, device=dev)
        if self.band_rows:
            nb = -(-n1 // self.band_rows)
            self.bands = [t.empty((self.W, nb, n2), dtype=t.int32, device=dev) for _ in range(nslots)]
            self.l16_ovf = t.zeros(1, dtype=t.int32, device=dev)
        self._pers_W = self.W
        self._pers_key = key
        self._graph = None

    def _band_rows(self) -> int:
        """Rows per band of hszg_band_scan (0: not applicable -> decode_rowscan + col_scan): whole tiles
        of 256 chunks, and enough bands that a window launches >= 8 CTAs per SM."""
        n1, n2 = self.sf.global_dims[1], self.sf.global_dims[2]
        if n2 % 32 or n2 > 4096:
            return 0
        rpt = 256 // (n2 // 32)
        if self.band_rows_req:
            return int(self.band_rows_req)
        # whole band_scan tiles where rpt is a multiple of 16 (multiples of 16 take the ring z-sweep,
        # zring.cu); otherwise 64 rows (the band's last tile is partial)
        unit = rpt if rpt >= 64 and rpt % 16 == 0 else 64
        want = -(-16 * _SMS // max(1, min(self.W, self.sf.nz)))
        br = -(-n1 // want)
        br = -(-br // unit) * unit
        if self.overlap:
            # persistent scans under the sweeps: the grid no longer needs many (band, plane) items,
            # and taller bands mean fewer band-offset rows (A) to write, prefix and re-read — up to
            # 256 rows while >= 2 items per SM remain (config 5: 64 -> 256 rows, step 56.1 -> 55.5 ms;
            # taller bands risk the int8 L range: 512 / 1024 gain < 0.1 ms more, 2048 overflows)
            cap = n1 * max(1, min(self.W, self.sf.nz)) // (2 * _SMS)
            br = max(br, min(256, cap) // unit * unit)
        return br

    def _stage_boundary(self):
        """Copy this run's halo / carry planes into the persistent buffers read by the loop."""
        self._persistent()
        if self.halo_lo is not None:
            self.halo_buf[0].copy_(self.halo_lo)
        if self.halo_hi is not None:
            self.halo_buf[1].copy_(self.halo_hi)
        if self.sf.kind == HSZP_ND and self.sf.z0 > 0 and self.carry is not None:
            self.carry_buf[0].copy_(self.carry)

    def _replay(self, outs):
        t = _lib.torch()
        key = tuple(0 if o is None else _lib.ptr(o) for o in outs) + (self.halo_lo is not None, self.halo_hi is not None,
                                                  self._emit_mode(), self.overlap, self.fused_layers, self.side_priority)
        if self._graph is None or self._graph_key != key:
            self._fused_loop(outs)                        # warm-up: workspaces, smem attributes
            t.cuda.synchronize()
            if self.timer is not None:
                self.timer.clear()                        # keep only the captured event nodes
            g = t.cuda.CUDAGraph()
            with t.cuda.graph(g):
                self._fused_loop(outs)
            self._graph, self._graph_key = g, key
        self._graph.replay()

    def _fused_loop(self, outs):
        _lib.call("hszg_acc_reset", _lib.ptr(self.acc), _lib.stream_handle())
        if self.sf.kind == HSZP_ND and self._one_pass_ok():
            self._run_lorenzo(outs)
        elif self.sf.kind == HSZP_ND:
            self._run_zsweep(outs)
        elif self._one_pass_ok():
            self._run_fused_blocks(outs)
        else:
            self._run_blocks(outs)

    one_pass = True             # HSZX_ND: one-pass decode + analytics kernel when eligible (fused.cu)
    # HSZP_ND one pass (lorenzo.cu): correct and tested, but slower than band scan + ring z-sweep so far
    lorenzo_one_pass = False
    fused_layers = FUSED_LAYERS

    def _one_pass_ok(self) -> bool:
        sf, ds = self.sf, self.ds
        n = sf.global_dims
        if not self.one_pass or not self._narrow_bw():
            return False
        if sf.kind == HSZP_ND:
            return self.lorenzo_one_pass and n[2] % 64 == 0 and n[2] <= 4096
        return (sf.kind == HSZX_ND and tuple(sf.block_dims) == (8, 8, 8)
                and sf.nz % 8 == 0 and n[1] % 8 == 0 and n[2] % 8 == 0)

    def _run_lorenzo(self, outs):
        """HSZP_ND in one pass over the slab (lorenzo.cu): a band-total pre-pass (hszg_band_scan with
        16-row bands, no L) then decode + x/y/z prefixes + gradient + Laplacian + stats in one kernel."""
        sf = self.sf
        if self.timer:
            self.timer.begin("prepass")
        err = _lib.Err()
        _lib.call("hszg_band_scan", ctypes.byref(self.ds.geom), ctypes.byref(self.ds.desc), 16, None,
                  _lib.ptr(self.lz_bands), _lib.ptr(self.lz_edges), 0, None, 0, _lib.stream_handle(), ctypes.byref(err),
                  err=err)
        if self.timer:
            self.timer.end("prepass", self._range_bytes(0, sf.nz) + self.lz_bands.numel() * 4 + self.lz_edges.numel() * 4)
            self.timer.begin("fused")
        carry = self.carry_buf[0] if sf.z0 > 0 else None
        upper = self.halo_buf[1] if self.halo_hi is not None else None
        outs_arr = self._outs_arr(outs, 0, self.sf.nz)
        _lib.call("hszg_lorenzo_onepass", ctypes.byref(self.ds.geom), ctypes.byref(self.ds.desc),
                  _lib.ptr(self.lz_bands), _lib.ptr(self.lz_edges), _lib.ptr(carry) if carry is not None else None,
                  _lib.ptr(upper) if upper is not None else None, sf.z0, sf.global_dims[0], outs_arr,
                  _lib.ptr(self.acc), self._emit_mode(), _lib.stream_handle(), ctypes.byref(err), err=err)
        if self.timer:
            self.timer.end("fused", self._range_bytes(0, sf.nz) + 16 * sf.nz * self.plane)

    def _run_fused_blocks(self, outs):
        """HSZX_ND in one launch over the whole slab: decode + gradient + Laplacian + stats, q never
        stored (fused.cu).  z segments of FUSED_LAYERS block layers per CTA column."""
        sf = self.sf
        nlay = sf.nz // 8
        if self.timer:
            self.timer.begin("fused")
        err = _lib.Err()
        outs_arr = self._outs_arr(outs, 0, self.sf.nz)
        _lib.call("hszg_fused_blocks", ctypes.byref(self.ds.geom), ctypes.byref(self.ds.desc), sf.z0,
                  sf.global_dims[0], _lib.ptr(self.halo_buf[0]) if self.halo_lo is not None else None,
                  _lib.ptr(self.halo_buf[1]) if self.halo_hi is not None else None, outs_arr, _lib.ptr(self.acc),
                  max(1, min(nlay, self.fused_layers)), self._emit_mode(), _lib.stream_handle(), ctypes.byref(err),
                  err=err)
        if self.timer:
            self.timer.end("fused", self._range_bytes(0, sf.nz) + 16 * sf.nz * self.plane)

    def _outs_arr(self, outs, a, b):
        """Output pointers of planes [a, b) (run() checked that all four exist)."""
        return (ctypes.c_void_p * 4)(*[_lib.ptr(o[a:b]) for o in outs])

    def _windows(self):
        nz = self.sf.nz
        return [(a, min(a + self.W, nz)) for a in range(0, nz, self.W)]

    def _run_blocks(self, outs):
        """HSZX_ND: k_tile_blocks decodes window k+2 while k_zgrad_lap (+ stats) runs on window k;
        three ring slots, halo planes by pointer (no copies)."""
        sf, ring = self.sf, self.ring
        n1, n2 = sf.global_dims[1], sf.global_dims[2]
        wins = self._windows()
        nw = len(wins)

        def decode(k):
            a, b = wins[k]
            if self.timer:
                self.timer.begin("reconstruct")
            self._decode_planes(a, b, ring[k % 3][: b - a])
            if self.timer:
                self.timer.end("reconstruct", self._range_bytes(a, b) + 4 * (b - a) * self.plane)

        decode(0)
        if nw > 1:
            decode(1)
        for k, (a, b) in enumerate(wins):
            if k > 0:
                pa, pb = wins[k - 1]
                prev = ring[(k - 1) % 3][pb - pa - 1]
            else:
                prev = self.halo_buf[0] if self.halo_lo is not None else None
            if k + 1 < nw:
                nxt = ring[(k + 1) % 3][0]
            else:
                nxt = self.halo_buf[1] if self.halo_hi is not None else None
            if self.timer:
                self.timer.begin("stencil")
            _lib.call("hszg_zgrad_lap", _lib.ptr(ring[k % 3]), n1, n2, 0, b - a, sf.z0 + a, sf.global_dims[0],
                      ctypes.c_double(sf.eps), self._outs_arr(outs, a, b), _lib.ptr(self.acc),
                      _lib.ptr(prev) if prev is not None else None, _lib.ptr(nxt) if nxt is not None else None,
                      self._emit_mode(), _lib.stream_handle())
            if self.timer:
                self.timer.end("stencil", (4 + 16) * (b - a) * self.plane)
            if k + 2 < nw:
                decode(k + 2)

    # HSZP_ND: band scans on a high-priority side stream, as a persistent grid beside the z-sweeps
    # (config 5: HSZP_ND op 32.5 -> 30.9 ms; bench.py --overlap 1, the default there); off by default
    # here so each kernel's event time is its own
    overlap = False
    side_priority = -1

    def _run_zsweep(self, outs):
        """HSZP_ND: band scan (decode + x / in-band y prefix) of window k, then the ring z-sweep of
        window k once window k+1 is decoded too (its first plane is the lookahead).  With `overlap`
        the band scans run on a side stream, NS = 3 ring slots ahead: scan k+2 overlaps sweep k,
        and scan k+3 waits for sweep k to release its slot (events; captured as graph edges)."""
        t = _lib.torch()
        sf, ring = self.sf, self.ring
        n1, n2 = sf.global_dims[1], sf.global_dims[2]
        wins = self._windows()
        nw = len(wins)
        ns = len(ring)
        br = self.band_rows
        l16 = bool(br) and ring[0].dtype == t.int16      # narrow L (int16 slots, int8 windows use half)
        modes = [self._l_mode(a) if l16 else 0 for a, _ in wins]
        self._l16_used = l16
        if l16:
            self.l16_ovf.zero_()
        main = t.cuda.current_stream()
        side = self._side_stream() if (self.overlap and ns >= 3) else main
        # on the side stream: a persistent scan grid (1 CTA per SM) that co-resides with the sweeps
        scan_ctas = 1 if side is not main else 0
        dec_done = [t.cuda.Event() for _ in range(nw)]
        sweep_done = [t.cuda.Event() for _ in range(nw)]

        def decode(k):
            a, b = wins[k]
            if self.timer:
                self.timer.begin("reconstruct")
            sub = self.ds.plane_view(a, b)
            err = _lib.Err()
            if br:
                _lib.call("hszg_band_scan", ctypes.byref(sub.geom), ctypes.byref(sub.desc), br,
                          _lib.ptr(ring[k % ns]), _lib.ptr(self.bands[k % ns]), None, modes[k],
                          _lib.ptr(self.l16_ovf) if l16 else None, scan_ctas, _lib.stream_handle(), ctypes.byref(err),
                          err=err)
            else:
                _lib.call("hszg_decode_rowscan", ctypes.byref(sub.geom), ctypes.byref(sub.desc),
                          _lib.ptr(ring[k % ns]), _lib.stream_handle(), ctypes.byref(err), err=err)
                _lib.call("hszg_col_scan", _lib.ptr(ring[k % ns]), b - a, n1, n2, _lib.stream_handle())
            if self.timer:
                self.timer.end("reconstruct", self._range_bytes(a, b) + (4, 2, 1)[modes[k]] * (b - a) * self.plane)

        issued = 0

        def issue_decodes(upto):
            nonlocal issued
            with t.cuda.stream(side):
                while issued <= min(upto, nw - 1):
                    k = issued
                    if k >= ns:
                        side.wait_event(sweep_done[k - ns])     # slot k % ns released by sweep k - ns
                    decode(k)
                    dec_done[k].record(side)
                    issued += 1

        if side is not main:
            fork = t.cuda.Event()
            fork.record(main)
            side.wait_event(fork)
        carry = self.carry_buf[0] if sf.z0 > 0 else None
        for k, (a, b) in enumerate(wins):
            issue_decodes(k + ns - 1 if side is not main else k + 1)
            if side is not main:
                main.wait_event(dec_done[min(k + 1, nw - 1)])
            look = ring[(k + 1) % ns][0] if k + 1 < nw else None
            upper = self.halo_buf[1] if (k + 1 == nw and self.halo_hi is not None) else None
            out_carry = self.carry_buf[1 + (k % 2)]
            if self.timer:
                self.timer.begin("stencil")
            _lib.call("hszg_zsweep_grad_lap", _lib.ptr(ring[k % ns]), n1, n2, b - a,
                      _lib.ptr(look) if look is not None else None, _lib.ptr(carry) if carry is not None else None,
                      _lib.ptr(upper) if upper is not None else None, _lib.ptr(out_carry), sf.z0 + a,
                      sf.global_dims[0], ctypes.c_double(sf.eps), self._outs_arr(outs, a, b), _lib.ptr(self.acc),
                      _lib.ptr(self.bands[k % ns]) if br else None,
                      _lib.ptr(self.bands[(k + 1) % ns]) if (br and look is not None) else None, br,
                      modes[k] | ((modes[k + 1] if k + 1 < nw else modes[k]) << 4), self._emit_mode(),
                      _lib.stream_handle())
            if self.timer:
                self.timer.end("stencil", ((4, 2, 1)[modes[k]] + 16) * (b - a) * self.plane)
            sweep_done[k].record(main)
            carry = out_carry
        if side is not main:
            main.wait_event(dec_done[nw - 1])                  # join the side stream

    def _side_stream(self):
        t = _lib.torch()
        if getattr(self, "_side", None) is None:
            # higher priority than the sweeps: the block scheduler places the persistent band-scan
            # CTAs first, one per SM beside two sweep CTAs (zring.cu: 64 registers, max carveout)
            self._side = t.cuda.Stream(priority=self.side_priority)
        return self._side

    def _finish_stats(self, _prepared):
        self.local_sums = self.acc
        if _prepared:
            return acc_to_ints(self.acc)
        ct = self.comm_timer if self.comm.world > 1 else None
        if ct:
            ct.begin("stats_allgather")
        parts = self.comm.all_gather(self.acc)
        if ct:
            ct.end("stats_allgather", 0)
        tot = dict(s1=0, s2=0, count=0, vmin=2**31, vmax=-(2**31))
        for p in parts:
            d = acc_to_ints(p)
            tot["s1"] += d["s1"]
            tot["s2"] += d["s2"]
            tot["count"] += d["count"]
            tot["vmin"] = min(tot["vmin"], d["vmin"])
            tot["vmax"] = max(tot["vmax"], d["vmax"])
        n = int(np.prod(self.sf.global_dims))
        mean, var = finalize_mean_var(tot["s1"], tot["s2"], n, self.sf.eps)
        return dict(mean=mean, var=var, **tot)

    # -- general loop (any geometry / output type) ------------------------------------------------
    @property
    def buf(self):
        if self._buf is None:
            t = _lib.torch()
            n1, n2 = self.sf.global_dims[1], self.sf.global_dims[2]
            self._buf = t.empty((self.W + self.G + 2, n1, n2), dtype=t.int32, device=_lib.device())
        return self._buf

    def _run_generic(self, outs, stats, _prepared):
        from . import device as devmod

        sf, buf, W, G = self.sf, self.buf, self.W, self.G
        nz = sf.nz
        if self.halo_lo is not None:
            buf[0].copy_(self.halo_lo)
        decoded = 0                                      # next local plane to decode
        for w, a in enumerate(range(0, nz, W)):
            b = min(a + W, nz)
            need = min(b + 1, nz)
            if decoded < need:
                e = min(nz, -(-need // G) * G)
                s = decoded
                if self.timer:
                    self.timer.begin("reconstruct")
                self._decode_planes(s, e, buf[s - a + 1:e - a + 1])
                if sf.kind == HSZP_ND:
                    carry = buf[s - a] if (s > 0 or sf.z0 > 0) else None
                    if s == 0 and sf.z0 > 0:
                        carry = self.carry
                    if carry is not None:
                        _lib.call("hszg_add_plane", _lib.ptr(buf[s - a + 1]), _lib.ptr(carry), self.plane,
                                  (e - s) * self.plane, _lib.stream_handle())
                if self.timer:
                    self.timer.end("reconstruct", self._range_bytes(s, e) + 4 * (e - s) * self.plane)
                decoded = e
            if b == nz and self.halo_hi is not None:
                buf[b - a + 1].copy_(self.halo_hi)
            if self.timer:
                self.timer.begin("stencil")
            devmod.stencil_window(_lib.OP_GRAD_LAP, [buf], [sf.eps], [o[a:b] for o in outs], 1, 1 + (b - a),
                                  sf.z0 + a - 1, sf.global_dims[0])
            if self.timer:
                self.timer.end("stencil", (4 + 4 * len(outs)) * (b - a) * self.plane)
            if stats and sf.kind == HSZP_ND:
                if self.timer:
                    self.timer.begin("stats")
                devmod.reduce_i32(buf[1:1 + (b - a)], out=self.win_sums[w * SUMS_BYTES:(w + 1) * SUMS_BYTES])
                if self.timer:
                    self.timer.end("stats", 4 * (b - a) * self.plane)
            if b < nz:                                   # slide: planes [b-1, decoded) to the front
                for k, z in enumerate(range(b - 1, decoded)):
                    buf[k].copy_(buf[z - a + 1])
        if not stats:
            return None
        if sf.kind == HSZP_ND:
            local = devmod.sums_combine(self.win_sums, self.nwin)
        else:
            if self.timer:
                self.timer.begin("stats")
            local = self.ds.reduce(3)                    # fused: sum q, sum q^2 from the bytes (no scatter)
            if self.timer:
                self.timer.end("stats", self._range_bytes(0, nz))
        self.local_sums = local
        if _prepared:
            return sums_to_ints(local)               # emulated rank: the caller combines
        tot = combine_rank_sums(self.comm, local)
        n = int(np.prod(sf.global_dims))
        mean, var = finalize_mean_var(tot["s1"], tot["s2"], n, sf.eps)
        return dict(mean=mean, var=var, **tot)


def _plane_prefix(U):
    """2-D inclusive prefix of an int32 plane (the Lorenzo inverse of a 2-D HSZP_ND stream)."""
    t = _lib.torch()
    n1, n2 = U.shape
    g = _lib.make_geom(HSZP_ND, (n1, n2), (min(8, n1), min(8, n2)), 1.0)
    out = t.empty((n1, n2), dtype=t.int32, device=_lib.device())
    ws = _lib.workspace(_lib.ws_bytes(g, None, _lib.WS_RECONSTRUCT, _lib.I32))
    err = _lib.Err()
    _lib.call("hszg_recorrelate", ctypes.byref(g), _lib.ptr(U), None, _lib.ptr(out), _lib.I32, _lib.ptr(ws),
              ws.numel(), _lib.stream_handle(), ctypes.byref(err), err=err)
    return out
