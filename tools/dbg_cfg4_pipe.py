"""Debug driver: config-4 API stencils then a whole-field WindowPipeline, synchronising between steps."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2603_25206_b200 as h
from paper_2603_25206_b200 import synthetic, pipeline as P
from paper_2603_25206_b200.analytics import fields
S = h.Stage
f = synthetic.config4_field()
kind = h.CompressorKind[sys.argv[1] if len(sys.argv) > 1 else "HSZX_ND"]
c = h.compress(f, kind, h.ErrorBound("rel", 1e-4))
d = c.device()
def step(name, fn):
    r = fn(); torch.cuda.synchronize(); print("ok", name, flush=True); return r
for i in range(3):
    step(f"api grad {i}", lambda: fields.compute_field_op(c, "derivative", S.QUANTIZED, out="torch", out_dtype=np.float32))
for i in range(3):
    step(f"api lap {i}", lambda: fields.compute_field_op(c, "laplacian", S.QUANTIZED, out="torch", out_dtype=np.float32))
sf = P.ShardedField(int(kind), c.eps, tuple(c.shape.dims), tuple(c.block_dims), 0, c.shape.dims[0], d)
outs = step("alloc", lambda: [torch.empty(tuple(c.shape.dims), dtype=torch.float32, device="cuda") for _ in range(4)])
step("zeros", lambda: torch.zeros(64, device="cuda"))
pipe = step("pipe", lambda: P.WindowPipeline(sf, window=64))
P.apply_settings(pipe, **dict(P.HEADLINE_SETTINGS, exact_fp32=True))
print(step("run", lambda: pipe.run(outs)))
