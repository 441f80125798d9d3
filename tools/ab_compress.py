"""A/B of the GPU compress paths at BASELINE config 4 (512^3) and config 5 slabs: the one-pass kernel
(csrc/compress.cu) vs the multi-kernel chain (HSZG_COMPRESS=chain), CUDA-event time per call (median of
N, the call's one host read-back included), plus a byte-identity check of the two containers.

    python tools/ab_compress.py [--reps 11] [--dims 512 512 512]
"""
import argparse
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2603_25206_b200 import compressors as C, synthetic  # noqa: E402
from paper_2603_25206_b200.grid import GridShape  # noqa: E402


def timed(fn, reps):
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        out = fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
        del out
    return statistics.median(ts)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=11)
    ap.add_argument("--dims", type=int, nargs="+", default=[512, 512, 512])
    args = ap.parse_args()
    dims = tuple(args.dims)
    f = torch.from_numpy(synthetic.config4_field(dims=dims).astype(np.float32)).cuda()
    eps = 1e-3 * float(f.max() - f.min())
    n = f.numel()
    for kind in C.CompressorKind:
        bd = C.resolve_block_dims(kind, GridShape(dims), None)
        one = lambda: C.compress_device(f, kind, eps, bd)  # noqa: E731
        ds1 = one()
        C._ONE_PASS = False
        ds2 = one()
        t_chain = timed(one, args.reps)
        C._ONE_PASS = True
        t_one = timed(one, args.reps)
        same = (ds1.payload_len == ds2.payload_len and
                torch.equal(ds1.payload[: ds1.payload_len], ds2.payload[: ds2.payload_len]) and
                torch.equal(ds1.offsets, ds2.offsets) and
                (ds1.metadata is None or torch.equal(ds1.metadata, ds2.metadata)))
        algo = 4 * n + ds1.payload_len + 8 * ds1.offsets.numel() + (4 * ds1.metadata.numel() if ds1.metadata is not None else 0)
        print(f"{kind.name:8s} chain {t_chain:7.3f} ms  one-pass {t_one:7.3f} ms  "
              f"({algo / t_one / 1e6:7.1f} GB/s algorithmic, {algo / t_one / 1e6 / 6532.9:.3f} of peak)  identical={same}",
              flush=True)


if __name__ == "__main__":
    main()
