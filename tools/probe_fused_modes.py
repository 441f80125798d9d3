"""Probe: hszg_fused_blocks on a whole config-4 HSZX_ND field (512^3) by emitter mode (0 fast, 1 fp64
conversions, 2 table) and output subset (all four, gradient, Laplacian), CUDA-event median times; the
API's layer count (fields._fused_layers) and a few alternatives.

    python tools/probe_fused_modes.py
"""
import ctypes
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
    import torch
    import paper_2603_25206_b200 as h
    from paper_2603_25206_b200 import _lib, synthetic
    from paper_2603_25206_b200.analytics import fields
    f = synthetic.config4_field()
    c = h.compress(f, h.CompressorKind.HSZX_ND, h.ErrorBound("rel", 1e-4))
    ds = c.device().validate()
    dims = tuple(c.shape.dims)
    print("max_bw", ds.desc.max_bitwidth, "api layers", fields._fused_layers(dims))
    outs = [torch.empty(dims, dtype=torch.float32, device="cuda") for _ in range(4)]
    sets = {"all4": outs, "grad": outs[:3] + [None], "lap": [None, None, None, outs[3]]}
    for zl in (fields._fused_layers(dims), 16, 8, 4):
        for mode in (0, 1, 2):
            for name, o in sets.items():
                if mode == 0 and name != "all4":
                    continue
                ptrs = (ctypes.c_void_p * 4)(*[None if x is None else _lib.ptr(x) for x in o])

                def run():
                    err = _lib.Err()
                    _lib.call("hszg_fused_blocks", ctypes.byref(ds.geom), ctypes.byref(ds.desc), 0, dims[0], None, None,
                              ptrs, None, zl, mode, _lib.stream_handle(), ctypes.byref(err), err=err)
                print(f"zl={zl:3d} mode={mode} {name:5s} {med_ms(run):.4f} ms", flush=True)


if __name__ == "__main__":
    main()
