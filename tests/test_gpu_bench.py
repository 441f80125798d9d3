"""bench.py end to end on the GPU: the single-rank line, and the multi-rank z-slab path (halo
planes, HSZP_ND carry, all-gathered exact statistics) run as 2 ranks sharing one GPU over gloo —
a plumbing check (its timing is meaningless): the global mean / variance must equal the
single-rank run's exactly."""

import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
ARGS = ["--dims", "96", "512", "512", "--steps", "1", "--warmup", "3", "--no-e2e", "--no-cpu", "--window", "32", "--rows"]


def _line(out: str) -> dict:
    return json.loads([x for x in out.splitlines() if x.startswith("{")][-1])


def test_bench_single_and_two_ranks():
    one = subprocess.run([sys.executable, "bench.py", *ARGS], cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert one.returncode == 0, one.stderr[-2000:]
    l1 = _line(one.stdout)
    assert l1["n_gpus"] == 1 and l1["value"] > 0 and l1["gpu_launches"] > 0
    env = dict(os.environ, HSZG_DIST_BACKEND="gloo")
    # bench.py --gpus 2 re-launches itself as 2 ranks (torch.distributed.run); here they share one GPU over gloo
    two = subprocess.run([sys.executable, "bench.py", "--gpus", "2", *ARGS], cwd=ROOT, capture_output=True,
                         text=True, timeout=900, env=env)
    assert two.returncode == 0, two.stderr[-3000:]
    l2 = _line(two.stdout)
    assert l2["n_gpus"] == 2 and l2["nccl"]["ranks"] == 2
    assert l2["stats_check"] == l1["stats_check"]
    for ln in (l1, l2):
        par = ln["parity"]
        assert par["exact_bit_exact"] and par["fast_within_tol"], par
        assert par["all_planes_hszp_nd_eq_hszx_nd"] and par["bit_exact_sums_across_kinds_and_emitters"], par
        assert par["rank0_container_decode_eq_quantize"], par
    assert "comm_ms_per_step" in l2 and l1["exact_fp32"]["ms_per_step"] > 0
