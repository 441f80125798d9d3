"""Host-side profile of one pipeline step (cProfile) + GPU kernel summary (torch.profiler)."""
import cProfile
import io
import pstats
import sys
import time

sys.path.insert(0, ".")
import torch

from paper_2603_25206_b200 import pipeline, synthetic
from paper_2603_25206_b200.quant import field_minmax

dims = tuple(int(x) for x in sys.argv[1:4]) if len(sys.argv) > 3 else (256, 2048, 2048)
field = synthetic.gen_config5_slab(0, dims[0], dims=dims)
lo, hi, _ = field_minmax(field.reshape(-1))
eps = 1e-3 * (hi - lo)
pipes = {}
for kind in (1, 3):
    sf = pipeline.compress_shard(field, kind, eps, (8, 8, 8), 0, dims[0], dims)
    pipes[kind] = pipeline.WindowPipeline(sf, pipeline.Comm(), 64)
del field
outs = [torch.empty(dims, dtype=torch.float32, device="cuda") for _ in range(4)]


def step():
    for k in (1, 3):
        pipes[k].run(outs)


step()
torch.cuda.synchronize()
for k in (1, 3):
    t0 = time.perf_counter()
    pipes[k].run(outs)
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    print(f"kind {k}: host loop {1e3*(t1-t0):.1f} ms, +sync {1e3*(t2-t1):.1f} ms")
pr = cProfile.Profile()
pr.enable()
step()
torch.cuda.synchronize()
pr.disable()
s = io.StringIO()
pstats.Stats(pr, stream=s).sort_stats("tottime").print_stats(25)
print(s.getvalue()[:6000])
