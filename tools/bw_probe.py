"""HBM ceiling for write-heavy streams: write-only (fill_), copy (1:1) and a 1-read : 4-write pattern."""
import torch

n = 1 << 30  # 4 GiB fp32
a = torch.empty(n, dtype=torch.float32, device="cuda")
bs = [torch.empty(n // 4, dtype=torch.float32, device="cuda") for _ in range(4)]
src = torch.randn(n // 4, device="cuda")
ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]


def timeit(fn, nbytes, reps=10):
    fn()
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(reps):
        ev[0].record()
        fn()
        ev[1].record()
        torch.cuda.synchronize()
        best = min(best, ev[0].elapsed_time(ev[1]))
    return nbytes / best / 1e6


print("write-only fill_      GB/s", round(timeit(lambda: a.fill_(1.0), 4 * n), 1))
print("copy 1:1              GB/s", round(timeit(lambda: a[: n // 2].copy_(a[n // 2:]), 4 * n), 1))
print("1 read : 4 writes     GB/s", round(timeit(lambda: torch.stack([src, src, src, src]), 4 * n // 4 * 5), 1))
