"""Generate golden fixtures by running the REAL reference package.

Run in the build container (where /root/reference exists):

    python tests/golden/make_golden.py

It imports ``hsz`` from /root/reference/pkg/src (read-only, never copied),
compresses seeded synthetic fields with every compressor kind and records the
reference's own outputs: container bytes, stage-② residuals, stage-③ indices,
mean/std at every stage, stencils at ②/③/④, divergence/curl, codec payload
digests and corruption messages.  The fixtures pin ``oracle/`` (CPU tests)
and, through the oracle, the CUDA path (GPU tests).  Output: golden.npz +
golden.json next to this script.
"""

from __future__ import annotations

import hashlib
import json
import os
import sys

import numpy as np

REF_SRC = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))


def main():
    sys.path.insert(0, REF_SRC)
    import hsz  # the reference
    from hsz import codec, io as hio
    from hsz.analytics import fields, stats
    from hsz.compressors import CompressorKind, compress
    from hsz.quant import ErrorBound
    from hsz.stages import Stage, partial_decompress

    sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
    from oracle.hsz_oracle import random_field

    arrays = {}
    index = {"reference_backend": hsz.kernel_backend, "cases": [], "vector": [], "codec": [],
             "errors": []}

    def put(key, value):
        arrays[key] = np.asarray(value)

    rng = np.random.default_rng(20240817)
    specs = []
    for dims in [(97,), (17, 13), (7, 6, 11), (40, 23), (12, 10, 9), (33, 65), (5, 9, 70)]:
        for kind in CompressorKind:
            if kind.is_nd and len(dims) < 2:
                continue
            specs.append((dims, kind, None))
    # non-default block geometries (edge blocks, multi-chunk and partial segments)
    specs += [((97,), CompressorKind.HSZX, (7,)), ((200,), CompressorKind.HSZP, (40,)),
              ((17, 13), CompressorKind.HSZX_ND, (3, 5)), ((12, 10, 9), CompressorKind.HSZX_ND, (4, 4, 3)),
              ((9, 20, 21), CompressorKind.HSZX_ND, (8, 8, 8)), ((40, 23), CompressorKind.HSZX, (70,))]
    example = np.array([[1.2, 1.5, -2.3, -2.5], [2.5, -1.0, 2.0, 1.7]], dtype=np.float32)

    cases = [("example", example, CompressorKind.HSZX_ND, ErrorBound("abs", 0.1), (2, 2))]
    for kind in CompressorKind:
        cases.append((f"example_{kind.cli_name}", example, kind, ErrorBound("abs", 0.1), None))
    for i, (dims, kind, bd) in enumerate(specs):
        texture = ("smooth", "noise", "mixed")[i % 3]
        field = random_field(rng, dims, texture)
        bound = ErrorBound("abs", 0.01) if i % 2 == 0 else ErrorBound("rel", 1e-3)
        cases.append((f"c{i}_{kind.cli_name}_{'x'.join(map(str, dims))}", field, kind, bound, bd))

    for name, field, kind, bound, bd in cases:
        c = compress(field, kind, bound, bd)
        blob = hio.stream_to_bytes(c)
        ds = partial_decompress(c, Stage.DECORRELATED)
        qf = partial_decompress(c, Stage.QUANTIZED)
        full = partial_decompress(c, Stage.FULL)
        entry = {"name": name, "kind": int(kind), "dims": list(field.shape),
                 "bound": [bound.mode, bound.requested],
                 "block_dims": None if bd is None else list(bd),
                 "resolved_block_dims": list(c.block_dims), "eps": c.eps, "stats": {}}
        put(f"{name}/field", field)
        put(f"{name}/container", np.frombuffer(blob, dtype=np.uint8))
        put(f"{name}/p", ds.values)
        put(f"{name}/q", qf.values)
        put(f"{name}/full", full)
        put(f"{name}/p_grid", ds.as_grid())
        stages = [Stage.DECORRELATED, Stage.QUANTIZED, Stage.FULL]
        if kind.is_block_mean:
            stages = [Stage.META] + stages
        for st in stages:
            for op in ("mean", "std"):
                if op == "std" and st == Stage.META:
                    continue
                if field.size < 2 and op == "std":
                    continue
                entry["stats"][f"{op}@{int(st)}"] = stats.compute_stat(c, op, st).value
        if field.ndim >= 2:
            st_list = [Stage.QUANTIZED, Stage.FULL] + ([Stage.DECORRELATED] if kind.is_nd else [])
            for st in st_list:
                d = fields.compute_field_op(c, "derivative", st)
                for ax, comp in enumerate(d.components):
                    put(f"{name}/deriv{int(st)}_{ax}", comp)
                lap = fields.compute_field_op(c, "laplacian", st)
                put(f"{name}/lap{int(st)}", lap.components[0])
        elif field.ndim == 1:
            d = fields.compute_field_op(c, "derivative", Stage.QUANTIZED)
            put(f"{name}/deriv3_0", d.components[0])
        if kind.is_nd and field.ndim >= 2:
            sd = fields.streamed_derivative(c)
            for ax, comp in enumerate(sd.components):
                put(f"{name}/streamed_{ax}", comp)
        index["cases"].append(entry)

    # vector operators
    vrng = np.random.default_rng(11)
    for dims in ((12, 13), (6, 7, 8)):
        for kind in (CompressorKind.HSZP_ND, CompressorKind.HSZX_ND):
            name = f"vec_{kind.cli_name}_{'x'.join(map(str, dims))}"
            comps = [random_field(vrng, dims) for _ in dims]
            srcs = tuple(compress(f, kind, ErrorBound("abs", 0.005)) for f in comps)
            for j, s in enumerate(srcs):
                put(f"{name}/container{j}", np.frombuffer(hio.stream_to_bytes(s), dtype=np.uint8))
            for st in (Stage.DECORRELATED, Stage.QUANTIZED, Stage.FULL):
                put(f"{name}/div{int(st)}", fields.divergence(srcs, st).components[0])
                for j, comp in enumerate(fields.curl(srcs, st).components):
                    put(f"{name}/curl{int(st)}_{j}", comp)
            index["vector"].append({"name": name, "kind": int(kind), "dims": list(dims)})

    # codec streams (test_kernels.py:_random_cases style + criterion 9), stored as digests
    crng = np.random.default_rng(20240817)
    for i in range(25):
        size = int(crng.integers(1, 2000))
        scale = int(crng.choice([1, 7, 2**10, 2**24, 2**30]))
        values = crng.integers(-scale, scale, size=size, endpoint=True).astype(np.int32)
        cut = int(crng.integers(0, size + 1))
        segments = [(0, cut), (cut, size)] if 0 < cut < size else [(0, size)]
        spans = codec.spans_from_segments(segments)
        payload, offsets = codec.encode_stream(values, spans)
        put(f"codec{i}/values", values)
        put(f"codec{i}/spans", spans)
        put(f"codec{i}/payload", np.frombuffer(payload, dtype=np.uint8))
        put(f"codec{i}/offsets", offsets)
        index["codec"].append(f"codec{i}")

    big = np.random.default_rng(53)
    n_chunks = 10**5
    counts = big.integers(1, 33, size=n_chunks)
    widths = big.integers(0, 32, size=n_chunks)
    scales = (np.int64(1) << widths) - 1
    values = np.concatenate([big.integers(-s, s, size=k, endpoint=True) if s else np.zeros(k, np.int64)
                             for k, s in zip(counts, scales)]).astype(np.int32)
    ends = np.cumsum(counts)
    spans = np.stack([ends - counts, ends], axis=1).astype(np.int64)
    payload, offsets = codec.encode_stream(values, spans)
    index["criterion9"] = {"seed": 53, "n_chunks": n_chunks,
                           "payload_sha256": hashlib.sha256(payload).hexdigest(),
                           "offsets_sha256": hashlib.sha256(offsets.astype("<u8").tobytes()).hexdigest(),
                           "payload_len": len(payload)}

    # corruption messages (the reference decoder's exact text)
    vals = np.arange(-40, 40, dtype=np.int32)
    spans = codec.spans_from_segments([(0, 80)])
    payload, offsets = codec.encode_stream(vals, spans)
    corrupt = {
        "truncated": payload[:-1],
        "bitwidth": bytes([40]) + payload[1:],
        "past_end": payload[: int(offsets[-1])],
        "neg_zero": bytes([1, 0b1, 0b0]),
    }
    for key, buf in corrupt.items():
        sp = spans if key != "neg_zero" else np.array([[0, 1]], dtype=np.int64)
        off = offsets if key != "neg_zero" else np.array([0], dtype=np.uint64)
        try:
            codec.decode_stream(buf, sp, off)
            msg = None
        except Exception as exc:  # noqa: BLE001 - recording the reference's behaviour
            msg = [type(exc).__name__, str(exc)]
        put(f"err_{key}/payload", np.frombuffer(buf, dtype=np.uint8))
        put(f"err_{key}/spans", sp)
        put(f"err_{key}/offsets", off)
        index["errors"].append({"name": f"err_{key}", "raises": msg})

    np.savez_compressed(os.path.join(HERE, "golden.npz"), **arrays)
    with open(os.path.join(HERE, "golden.json"), "w") as fh:
        json.dump(index, fh, indent=1, sort_keys=True)
    print(f"wrote {len(arrays)} arrays, {len(index['cases'])} cases")


if __name__ == "__main__":
    main()
