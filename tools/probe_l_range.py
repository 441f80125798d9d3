"""Probe: range of the HSZP_ND band-local prefixes L (hszg_band_scan, int32) of the config-5 field by band
height — could they be stored in 4 bits?  Planes [1, 65) of a 2048^2 x 80 slab (plane 0's L is q itself).

    python tools/probe_l_range.py
"""
import ctypes
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch
    from paper_2603_25206_b200 import _lib, pipeline as P, synthetic
    dims = (80, 2048, 2048)
    f = synthetic.gen_config5_slab(0, 80)
    eps = 0.004426495552062988     # the bench's global absolute bound (rel 1e-3 of the field's range)
    sf = P.compress_shard(f, P.HSZP_ND, eps, (8, 8, 8), 0, dims[0], dims)
    ds = sf.ds.validate()
    sub = ds.plane_view(0, 72)
    for br in (16, 32, 64, 128, 256):
        nb = -(-dims[1] // br)
        L = torch.empty((72, dims[1], dims[2]), dtype=torch.int32, device="cuda")
        A = torch.empty((72, nb, dims[2]), dtype=torch.int32, device="cuda")
        err = _lib.Err()
        _lib.call("hszg_band_scan", ctypes.byref(sub.geom), ctypes.byref(sub.desc), br, _lib.ptr(L), _lib.ptr(A), None,
                  0, None, 0, _lib.stream_handle(), ctypes.byref(err), err=err)
        Lr = L[1:]
        h = torch.histc(Lr.float().clamp(-16, 16), bins=33, min=-16.5, max=16.5)
        frac4 = float(((Lr >= -8) & (Lr <= 7)).float().mean())
        print(f"band_rows={br:4d} L min {int(Lr.min())} max {int(Lr.max())}  in [-8,7]: {frac4:.6f}  "
              f"A min {int(A[1:].min())} max {int(A[1:].max())}", flush=True)


if __name__ == "__main__":
    main()
