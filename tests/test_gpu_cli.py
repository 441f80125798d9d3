"""The GPU CLI (paper_2603_25206_b200/cli.py) against the reference CLI's contract
(cli.py:71-231; scenarios of pkg/tests/test_cli.py restated): key=value output, file formats, exit
codes, the applicability matrix, and the cost-aware ``--stage auto`` (identical results to the
reference's automatic stage, fewer GPU bytes)."""

import numpy as np
import pytest

from oracle import hsz_oracle as O

pytestmark = pytest.mark.gpu


@pytest.fixture
def run():
    from click.testing import CliRunner

    from paper_2603_25206_b200.cli import main

    r = CliRunner()
    return lambda args: r.invoke(main, [str(a) for a in args])


def _kv(out):
    return dict(line.partition("=")[::2] for line in out.strip().splitlines() if "=" in line)


def _compress(run, tmp_path, field, kind, bound, block=None, name="y"):
    raw, out = tmp_path / f"{name}.f32", tmp_path / f"{name}.hsz"
    np.asarray(field, dtype="<f4").tofile(raw)
    args = ["compress", "--input", raw, "--dims", ",".join(map(str, field.shape)), "--compressor", kind,
            "--error", bound, "--output", out]
    if block:
        args += ["--block", block]
    r = run(args)
    assert r.exit_code == 0, r.output
    return r, out


def test_cli_worked_example(run, tmp_path, example_field):
    r, out = _compress(run, tmp_path, example_field, "hszx-nd", "abs:0.1", "2,2")
    kv = _kv(r.output)
    assert kv["eps"] == "0.1" and float(kv["ratio"]) > 0
    ref = O.compress(example_field, 3, "abs", 0.1, (2, 2))
    assert out.read_bytes() == O.stream_to_bytes(ref)
    for stage, want, dt in (("meta", [5, -1], "<i4"), ("decorrelated", [1, 3, 8, -10, -10, -11, 11, 10], "<i4"),
                            ("quantized", [6, 8, 13, -5, -11, -12, 10, 9], "<i4")):
        p = tmp_path / f"{stage}.bin"
        assert run(["decompress", "--input", out, "--stage", stage, "--output", p]).exit_code == 0
        assert np.fromfile(p, dtype=dt).tolist() == want
    full = tmp_path / "d.f32"
    assert run(["decompress", "--input", out, "--stage", "full", "--output", full]).exit_code == 0
    assert np.abs(np.fromfile(full, dtype="<f4").reshape(2, 4) - example_field).max() <= 0.1 + 1e-6
    assert _kv(run(["analyze", "--op", "std", "--input", out, "--stage", "decorrelated"]).output)["std"] == "2"
    r = run(["analyze", "--op", "mean", "--input", out, "--stage", "auto", "--explain"])
    assert _kv(r.output)["mean"] == "0.4" and _kv(r.output)["stage"] == "meta"
    info = _kv(run(["info", "--input", out]).output)
    assert (info["kind"], info["dims"], info["block"], info["n"], info["metadata"]) == ("hszx-nd", "2,4", "2,2", "8", "2")


def test_cli_relative_bound_eps(run, tmp_path, example_field):
    r, _ = _compress(run, tmp_path, example_field, "hszx-nd", "rel:0.02", "2,2")
    assert _kv(r.output)["eps"] == "0.1"


@pytest.mark.parametrize("kind", ["hszp-nd", "hszx-nd"])
def test_cli_auto_stage_cost_aware(run, tmp_path, rng, kind):
    """auto picks stage 3 for the nd stencils on the GPU (the reference picks 2: same integers, the GPU
    stage-2 path recorrelates first) — the written components are bit-identical to stage 2's."""
    f = O.random_field(rng, (16, 12))
    _, out = _compress(run, tmp_path, f, kind, "abs:0.01")
    r = run(["analyze", "--op", "derivative", "--input", out, "--output", tmp_path / "a", "--explain"])
    assert r.exit_code == 0, r.output
    kv = _kv(r.output)
    assert kv["stage"] == "quantized" and float(kv["cost_quantized"]) < float(kv["cost_decorrelated"])
    r2 = run(["analyze", "--op", "derivative", "--input", out, "--stage", "decorrelated", "--output", tmp_path / "b"])
    assert r2.exit_code == 0
    c = O.stream_from_bytes(out.read_bytes())
    want = O.derivative_q(O.stage3(c), c.eps)
    for name, w in zip(("dx", "dy"), want):
        a = np.fromfile(tmp_path / f"a.{name}.f32", dtype="<f4")
        b = np.fromfile(tmp_path / f"b.{name}.f32", dtype="<f4")
        assert np.array_equal(a, b) and np.array_equal(a, w.astype(np.float32).ravel())


def test_cli_divergence_and_errors(run, tmp_path, rng):
    paths = [str(_compress(run, tmp_path, O.random_field(rng, (10, 10)), "hszx-nd", "abs:0.01", name=n)[1])
             for n in ("u", "v")]
    r = run(["analyze", "--op", "divergence", "--u", paths[0], "--v", paths[1], "--output", tmp_path / "field"])
    assert r.exit_code == 0, r.output and (tmp_path / "field.div.f32").exists()
    _, out = _compress(run, tmp_path, O.random_field(rng, (64,)), "hszp", "abs:0.01", name="one")
    r = run(["analyze", "--op", "derivative", "--input", out, "--stage", "decorrelated"])
    assert r.exit_code == 1 and "applicability" in (r.output + (r.stderr if r.stderr_bytes else ""))
    r = run(["compress", "--input", "/nonexistent", "--dims", "4", "--compressor", "hszp", "--error", "abs:0.1",
             "--output", tmp_path / "x"])
    assert r.exit_code == 2
