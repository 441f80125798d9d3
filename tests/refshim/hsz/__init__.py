"""Test-side alias shim (TEST INFRASTRUCTURE, never imported by the product package): makes
``import hsz`` resolve to the drop-in ``paper_2603_25206_b200`` so the reference's own test files
(/root/reference/pkg/tests) import and run against it unchanged.

The two test-visible modules the drop-in does not ship come from the oracle:
* ``hsz.oracle`` — the float-domain textbook oracle (oracle.py:14-86, restated in oracle/hsz_oracle.py);
* ``hsz._kernels._fallback`` — the numpy byte-format oracle (_fallback.py:22-107: encode / decode /
  chunk_byte_size), here the oracle's C restatement;
and ``hsz._kernels._bitpack`` (the reference's optional compiled backend, test_kernels.py:9-16) is the
drop-in's CUDA plugin, so test_kernels.py compares the GPU codec against the byte-format oracle.
"""

import importlib
import os
import sys
import types

_ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
if _ROOT not in sys.path:
    sys.path.insert(0, _ROOT)

import numpy as _np  # noqa: E402

import paper_2603_25206_b200 as _pkg  # noqa: E402
from oracle import hsz_oracle as _O  # noqa: E402
from paper_2603_25206_b200 import *  # noqa: E402,F401,F403

kernel_backend = _pkg.kernel_backend

for _name in ("codec", "compressors", "counters", "errors", "grid", "io", "quant", "stages", "analytics",
              "analytics.stats", "analytics.fields", "analytics.regions", "_kernels", "cli"):
    _mod = importlib.import_module(f"paper_2603_25206_b200.{_name}")
    sys.modules[f"hsz.{_name}"] = _mod
    if "." not in _name:
        globals()[_name] = _mod

_oracle = types.ModuleType("hsz.oracle")
for _n in ("oracle_stats", "oracle_derivative", "oracle_laplacian", "oracle_divergence", "oracle_curl"):
    setattr(_oracle, _n, getattr(_O, _n))
sys.modules["hsz.oracle"] = _oracle
oracle = _oracle


def _spans(starts, ends):
    return _np.stack([_np.asarray(starts, dtype=_np.int64), _np.asarray(ends, dtype=_np.int64)], axis=1)


_fb = types.ModuleType("hsz._kernels._fallback")
_fb.chunk_byte_size = _O.chunk_byte_size
_fb.encode_stream = lambda values, starts, ends: _O.encode_stream(values, _spans(starts, ends))
_fb.decode_stream = lambda payload, starts, ends, offsets: _O.decode_stream(payload, _spans(starts, ends), offsets)
sys.modules["hsz._kernels._fallback"] = _fb
sys.modules["hsz._kernels"]._fallback = _fb
sys.modules["hsz._kernels._bitpack"] = sys.modules["hsz._kernels"]
