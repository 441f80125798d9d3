"""CPU tests of the C-ABI boundary and host-side logic (no GPU needed).

* libhszg.so loads and exports every entry point declared in include/hszg.h;
* the closed-form chunk geometry (csrc/common.cuh, exposed on the host via
  hszg_locate_chunks) reproduces the reference's span construction
  (compressors.segment_bounds + codec.spans_from_segments) for every kind;
* the product path refuses to run without a device (no CPU fallback).
"""

import ctypes
import os
import re

import numpy as np
import pytest

from oracle import hsz_oracle as O
from paper_2603_25206_b200 import _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared_symbols():
    with open(os.path.join(ROOT, "include", "hszg.h")) as fh:
        text = fh.read()
    return sorted(set(re.findall(r"^\s*(?:int|size_t|const char\*)\s+(hszg_\w+)\s*\(", text, flags=re.M)))


def test_library_exports_every_declared_symbol():
    lib = _lib.load_library()
    declared = _declared_symbols()
    assert len(declared) >= 30
    for name in declared:
        assert hasattr(lib, name), name
        assert isinstance(getattr(lib, name), ctypes._CFuncPtr)
    assert set(declared) <= set(_lib.EXPORTED_SYMBOLS), set(declared) - set(_lib.EXPORTED_SYMBOLS)
    assert lib.hszg_version().startswith(b"hszg")


def test_struct_layouts():
    assert ctypes.sizeof(_lib.Sums) == 64
    assert ctypes.sizeof(_lib.Err) == 4 + 4 + 8 * 3 + 192
    assert ctypes.sizeof(_lib.Geom) == 4 + 4 + 24 + 24 + 8 + 24 + 72


def _cases():
    rng = np.random.default_rng(3)
    out = [(3, (17, 13), (3, 5)), (1, (7, 6, 11), (8, 8, 8)), (0, (97,), (32,)), (2, (97,), (7,)),
           (3, (12, 10, 9), (4, 4, 3)), (1, (33, 65), (8, 8)), (2, (40, 23), (70,)), (3, (9, 20, 21), (8, 8, 8)),
           (3, (2, 4), (2, 2)), (0, (1,), (1,)), (3, (5, 9, 70), (8, 8, 8)), (1, (100, 500, 50), (8, 8, 8))]
    for _ in range(40):
        nd = int(rng.integers(1, 4))
        dims = tuple(int(rng.integers(1, 40)) for _ in range(nd))
        kind = int(rng.integers(0, 4))
        if kind in (1, 3) and nd < 2:
            kind -= 1
        bd = tuple(int(rng.integers(1, 12)) for _ in range(nd))
        out.append((kind, dims, bd))
    return out


@pytest.mark.parametrize("kind,dims,bd", _cases())
def test_closed_form_geometry_matches_reference_spans(kind, dims, bd):
    rbd = O.resolve_block_dims(kind, dims, bd if O.is_nd(kind) else (bd[0],))
    g = _lib.make_geom(kind, dims, rbd, 0.1)
    spans = O.stream_spans(kind, dims, rbd)
    assert int(g.n_chunks) == len(spans)
    st, en, seg = _lib.locate_chunks(g)
    assert np.array_equal(st, spans[:, 0]) and np.array_equal(en, spans[:, 1])
    if O.is_block_mean(kind):
        gd, gb = O.effective_geometry(kind, dims, rbd)
        assert int(g.n_blocks) == len(O.block_sizes(gd, gb))
        # segment id of every chunk = the block whose metadata it uses
        sizes = O.block_sizes(gd, gb)
        owner = np.repeat(np.arange(len(sizes)), sizes)
        assert np.array_equal(seg, owner[spans[:, 0]])


def test_geometry_rejects_bad_blocks():
    with pytest.raises(ValueError):
        _lib.make_geom(3, (4, 4), (5, 2), 0.1)
    with pytest.raises(ValueError):
        _lib.make_geom(1, (16,), (8,), 0.1)


def test_large_geometry_is_64bit():
    g = _lib.make_geom(1, (2048, 2048, 2048), (8, 8, 8), 1e-3)
    assert int(g.n) == 2048**3
    assert int(g.n_chunks) == 2048 * (2048 * 2048 // 32)
    g = _lib.make_geom(3, (2048, 2048, 2048), (8, 8, 8), 1e-3)
    assert int(g.n_chunks) == 256**3 * 16
    st, en, _ = _lib.locate_chunks(g, int(g.n_chunks) - 3, 3)
    assert en[-1] == 2048**3


def test_product_path_fails_loudly_without_cuda():
    import torch

    if torch.cuda.is_available():
        pytest.skip("a device is present")
    from paper_2603_25206_b200 import BackendUnavailableError, CompressorKind, ErrorBound, compress

    with pytest.raises(BackendUnavailableError):
        compress(np.zeros((4, 4), np.float32), CompressorKind.HSZP, ErrorBound("abs", 0.1))
