"""NVTX ranges per stage / operation (the reference's per-stage decode counters become
profiler ranges on the GPU path).  Each public entry point of the hot path is wrapped in a range
named "hsz/<op>" so an nsys / ncu --nvtx capture attributes every kernel to the API call and stage
that launched it.  Costs one push / pop (~1 us) per call; a no-op without CUDA.
"""

from __future__ import annotations

import functools


def ranged(name: str):
    def deco(fn):
        @functools.wraps(fn)
        def wrapper(*args, **kwargs):
            nv = _nvtx()
            if nv is None:
                return fn(*args, **kwargs)
            label = name
            stage = kwargs.get("stage", args[1] if len(args) > 1 and name.endswith(("decompress", "stat", "field_op"))
                               else None)
            if stage is not None and hasattr(stage, "name"):
                label = f"{name}[{stage.name.lower()}]"
            nv.range_push(label)
            try:
                return fn(*args, **kwargs)
            finally:
                nv.range_pop()
        return wrapper
    return deco


_NV = None


def _nvtx():
    global _NV
    if _NV is None:
        try:
            import torch

            _NV = torch.cuda.nvtx if torch.cuda.is_available() else False
        except Exception:  # noqa: BLE001
            _NV = False
    return _NV or None
