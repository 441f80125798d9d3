"""Out-of-core slab streaming: decode a container that stays in host memory.

The reference iterates slabs of a container it holds in host memory (``slab_iter`` /
``sliding_window``, stages.py:173-258; the paper's Algorithm 3, a 3-slab window for fields larger
than memory).  Here the container stays in pinned host memory and only the bytes of the slabs
being decoded live on the device:

* consecutive slabs are grouped into fetch units of at most ``budget`` container bytes (at least
  one slab); a unit is one contiguous chunk range — payload bytes, index entries and block means
  (chunks restart at every segment, compressors.py:105-119);
* units are copied host -> device on a copy stream into two device slots, unit k+1 while unit k
  decodes (CUDA events order slot reuse and first use);
* each unit is validated on the device once (the reference decoder's per-chunk checks,
  _bitpack.pyx:110-140) and every slab of it is a ``DeviceStream`` view whose payload pointer is
  shifted by the unit's first byte, so the container's absolute chunk offsets address the slot.

No whole-container upload happens: ``CompressedStream.device()`` is never called.
"""

from __future__ import annotations

import numpy as np

from . import _lib
from .compressors import CompressedStream, CompressorKind
from .device import DeviceStream

DEFAULT_BUDGET = 256 << 20      # container bytes per fetch unit


class HostSlabSource:
    """Streams the slabs ``bounds`` (axis-0 ranges, stages.slab_bounds) of a host container."""

    def __init__(self, c: CompressedStream, bounds, layout, budget: int = DEFAULT_BUDGET):
        t = _lib.torch()
        self.c = c
        self.bounds = list(bounds)
        self.layout = layout                      # (lo, hi) -> (first, last, meta_lo, meta_hi, dims, bd)
        payload = c.payload
        self.plen = len(payload)
        # pinned host copies of the container sections, kept on the stream object for later passes
        key = (id(payload), id(c._chunk_offsets), id(c._metadata))
        pin = getattr(c, "_pinned", None)
        if pin is None or pin[0] != key:
            h_payload = c.pinned_payload()                    # read_compressed: the file buffer itself
            if h_payload is None:
                h_payload = t.empty(max(self.plen, 1), dtype=t.uint8, pin_memory=True)
                if self.plen:
                    h_payload[: self.plen].copy_(t.frombuffer(bytearray(payload), dtype=t.uint8))
            offs = np.ascontiguousarray(np.asarray(c.chunk_offsets, dtype=np.uint64)).view(np.int64).copy()
            meta = c.metadata
            h_meta = None if meta is None else t.from_numpy(np.ascontiguousarray(meta, dtype=np.int32)).pin_memory()
            pin = (key, h_payload, offs, t.from_numpy(offs).pin_memory(), h_meta)
            c._pinned = pin
        _, self.h_payload, offs, self.h_offsets, self.h_meta = pin
        self.offs = offs
        self.nc = len(offs)
        # per slab: chunk range, absolute byte range, metadata range
        self.slabs = []
        for lo, hi in self.bounds:
            first, last, mlo, mhi, dims, bd = layout(lo, hi)
            b0 = int(offs[first]) if first < self.nc else self.plen
            b1 = int(offs[last]) if last < self.nc else self.plen
            self.slabs.append((first, last, b0, b1, mlo, mhi, dims, bd))
        # fetch units: consecutive slabs up to `budget` bytes
        self.units = []
        k = 0
        while k < len(self.slabs):
            j = k + 1
            while j < len(self.slabs) and self.slabs[j][3] - self.slabs[k][2] <= budget:
                j += 1
            self.units.append((k, j))
            k = j
        self.unit_of = np.empty(len(self.slabs), dtype=np.int64)
        for u, (a, b) in enumerate(self.units):
            self.unit_of[a:b] = u
        # two device slots sized for the largest unit
        dev = _lib.device()
        mb = mc = mm = 1
        for a, b in self.units:
            f0, _, b0, _, m0, _, _, _ = self.slabs[a]
            _, l1, _, e1, _, m1, _, _ = self.slabs[b - 1]
            mb = max(mb, e1 - (b0 & ~15))
            mc = max(mc, l1 - f0 + 1)
            mm = max(mm, m1 - m0)
        self.d_payload = [t.zeros(mb + 16 + _lib.PAYLOAD_PAD, dtype=t.uint8, device=dev) for _ in range(2)]
        self.d_offsets = [t.empty(mc, dtype=t.int64, device=dev) for _ in range(2)]
        self.d_meta = [t.empty(mm, dtype=t.int32, device=dev) for _ in range(2)] if self.h_meta is not None else None
        self.copy_stream = t.cuda.Stream()
        self.ready = [t.cuda.Event() for _ in range(2)]
        self.free = [t.cuda.Event() for _ in range(2)]
        self.slot_used = [False, False]
        self.fetched = {}                           # unit -> slot
        self.validated = {}                         # unit -> (canonical, max_bw)
        self.h2d_bytes = 0

    # ---- transfers --------------------------------------------------------------------
    def fetch(self, u: int):
        """Issue the H2D copy of unit u into slot u % 2 (asynchronous, copy stream)."""
        if u >= len(self.units) or u in self.fetched:
            return
        t = _lib.torch()
        s = u % 2
        a, b = self.units[u]
        first, _, b0, _, mlo, _, _, _ = self.slabs[a]
        _, last, _, e1, _, mhi, _, _ = self.slabs[b - 1]
        base = b0 & ~15
        with t.cuda.stream(self.copy_stream):
            if self.slot_used[s]:
                self.copy_stream.wait_event(self.free[s])      # the slot's previous unit is decoded
            nb = e1 - base
            if nb > 0:
                self.d_payload[s][:nb].copy_(self.h_payload[base:e1], non_blocking=True)
            ni = min(last + 1, self.nc) - first
            if ni > 0:
                self.d_offsets[s][:ni].copy_(self.h_offsets[first:first + ni], non_blocking=True)
            if self.d_meta is not None and mhi > mlo:
                self.d_meta[s][: mhi - mlo].copy_(self.h_meta[mlo:mhi], non_blocking=True)
            self.ready[s].record(self.copy_stream)
        self.h2d_bytes += (e1 - base) + 8 * max(0, min(last + 1, self.nc) - first) + 4 * max(0, mhi - mlo)
        self.slot_used[s] = True
        self.fetched = {k: v for k, v in self.fetched.items() if v != s}
        self.fetched[u] = s

    def release(self, u: int):
        """Mark unit u's slot reusable once the work queued so far on the compute stream is done."""
        s = self.fetched.get(u)
        if s is not None:
            self.free[s].record(_lib.torch().cuda.current_stream())

    # ---- views ------------------------------------------------------------------------
    def _view(self, s: int, u: int, a: int, b: int, dims, bd) -> DeviceStream:
        """DeviceStream over slabs [a, b) of unit u in slot s (absolute offsets, shifted payload)."""
        ua, _ = self.units[u]
        ufirst, _, ub0, _, umlo, _, _, _ = self.slabs[ua]
        first, _, _, _, mlo, _, _, _ = self.slabs[a]
        _, last, _, e1, _, mhi, _, _ = self.slabs[b - 1]
        offs = self.d_offsets[s][first - ufirst:last - ufirst]
        meta = None if self.d_meta is None else self.d_meta[s][mlo - umlo:mhi - umlo]
        sub = DeviceStream(int(self.c.kind), dims, bd, self.c.eps, self.d_payload[s], e1, offs, meta)
        sub.desc.payload = _lib.ptr(self.d_payload[s]) - (ub0 & ~15)   # absolute offset o -> slot byte
        sub.desc.payload_len = e1                                        # absolute end of the range
        return sub

    def slab(self, k: int) -> tuple:
        """(validated DeviceStream view of slab k, chunk count, payload bytes); prefetches the next unit."""
        t = _lib.torch()
        u = int(self.unit_of[k])
        self.fetch(u)
        s = self.fetched[u]
        a, b = self.units[u]
        t.cuda.current_stream().wait_event(self.ready[s])
        if u not in self.validated:
            lo, hi = self.bounds[a][0], self.bounds[b - 1][1]
            _, _, _, _, _, _, dims, bd = self.slabs[a]
            udims, ubd = self.unit_dims(lo, hi, dims, bd)
            whole = self._view(s, u, a, b, udims, ubd).validate()
            self.validated[u] = (int(whole.desc.canonical), int(whole.desc.max_bitwidth))
            self.fetch(u + 1)                        # overlap the next unit's copy with this one's decode
        first, last, b0, b1, _, _, dims, bd = self.slabs[k]
        sub = self._view(s, u, k, k + 1, dims, bd)
        sub.desc.canonical, sub.desc.max_bitwidth = self.validated[u]
        sub.validated = True
        return sub, last - first, b1 - b0, u

    def span(self, k0: int, k1: int) -> DeviceStream:
        """Validated DeviceStream view of slabs [k0, k1) of one unit (slab_iter decodes them together)."""
        sub0, _, _, u = self.slab(k0)
        if k1 == k0 + 1:
            return sub0
        assert int(self.unit_of[k1 - 1]) == u, "a span must stay inside one fetch unit"
        s = self.fetched[u]
        _, _, _, _, _, _, dims, bd = self.slabs[k0]
        sdims, sbd = self.unit_dims(self.bounds[k0][0], self.bounds[k1 - 1][1], dims, bd)
        sub = self._view(s, u, k0, k1, sdims, sbd)
        sub.desc.canonical, sub.desc.max_bitwidth = self.validated[u]
        sub.validated = True
        return sub

    def unit_dims(self, lo, hi, dims, bd):
        if self.c.kind.is_nd:
            return (hi - lo,) + tuple(self.c.shape.dims[1:]), tuple(
                min(b, n) for b, n in zip(self.c.block_dims, (hi - lo,) + tuple(self.c.shape.dims[1:])))
        return (hi - lo,), (min(self.c.block_dims[0], hi - lo),)


def should_stream(c: CompressedStream, from_host) -> bool:
    """from_host=None: stream when the container is not on the device yet and is larger than
    HSZG_DEVICE_BUDGET bytes (default: half the free device memory)."""
    if from_host is not None:
        return bool(from_host)
    if c._device is not None or c._payload is None:
        return False
    import os

    t = _lib.torch()
    budget = os.environ.get("HSZG_DEVICE_BUDGET")
    if budget is None:
        free, _ = t.cuda.mem_get_info()
        budget = free // 2
    size = len(c._payload) + 8 * len(c._chunk_offsets) + (0 if c._metadata is None else 4 * len(c._metadata))
    return size > int(budget)


__all__ = ["HostSlabSource", "should_stream", "DEFAULT_BUDGET", "CompressorKind"]
