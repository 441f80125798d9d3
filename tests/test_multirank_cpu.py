"""Multi-process CPU tests (gloo, world size 2) of the sharded pipeline's host-side logic.

The collectives of pipeline.py (halo exchange, all-gather of slab totals for the
HSZP_ND Lorenzo carry, exact int128 statistics combination) are exercised with
CPU tensors over gloo; the per-rank inputs (slab-total planes, boundary planes,
per-rank exact sums) come from the oracle, and the combined results are checked
against the oracle on the whole field.  No GPU needed.
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import hsz_oracle as O


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, result_queue):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2603_25206_b200 import pipeline

        comm = pipeline.Comm()
        assert comm.rank == rank and comm.world == world
        rng = np.random.default_rng(5)
        field = O.random_field(rng, (32, 12, 10), "smooth")
        eps = 0.01
        c = O.compress(field, O.HSZP_ND, "abs", eps, (8, 8, 8))
        q = O.stage3(c)
        p = O.stage2(c).reshape(q.shape).astype(np.int64)
        z0, z1 = pipeline.shard_planes(32, world, rank, 16)
        # HSZP_ND carry: T_g = P2(sum_{z in slab} p[z]); C_g = sum_{g'<g} T_g' == q[z0-1]
        U = p[z0:z1].sum(axis=0)
        T = np.cumsum(np.cumsum(U, axis=0), axis=1).astype(np.int64)
        T32 = ((T + 2**31) % 2**32 - 2**31).astype(np.int32)
        gathered = comm.all_gather(torch.from_numpy(T32))
        C = pipeline.exclusive_plane_prefix(gathered, rank).numpy()
        want_C = q[z0 - 1] if z0 > 0 else np.zeros_like(q[0])
        ok_carry = np.array_equal(C, want_C)
        # halo exchange: lower neighbour's last plane, upper neighbour's first plane
        lo, hi = comm.exchange(torch.from_numpy(q[z0].copy()), torch.from_numpy(q[z1 - 1].copy()),
                               torch.from_numpy(q[z0].copy()))
        ok_halo = (lo is None or np.array_equal(lo.numpy(), q[z0 - 1])) and (
            hi is None or np.array_equal(hi.numpy(), q[z1]))
        # exact statistics: int128 records combined across ranks (values above 2^64 on purpose)
        import ctypes

        from paper_2603_25206_b200 import _lib

        s = _lib.Sums()
        big1 = (3 + rank) * 2**70 + rank
        big2 = 2**100 + 7 * rank
        s.s1_lo, s.s1_hi = big1 & (2**64 - 1), big1 >> 64
        s.s2_lo, s.s2_hi = big2 & (2**64 - 1), big2 >> 64
        s.count = 10 + rank
        s.vmin, s.vmax = -rank, rank
        buf = torch.frombuffer(bytearray(ctypes.string_at(ctypes.addressof(s), 64)), dtype=torch.uint8)
        tot = pipeline.combine_rank_sums(comm, buf)
        want1 = sum((3 + r) * 2**70 + r for r in range(world))
        want2 = sum(2**100 + 7 * r for r in range(world))
        ok_sums = tot["s1"] == want1 and tot["s2"] == want2 and tot["count"] == sum(10 + r for r in range(world))
        ok_sums &= tot["vmin"] == -(world - 1) and tot["vmax"] == world - 1
        mm = torch.tensor([float(field[z0:z1].min()), -float(field[z0:z1].max())], dtype=torch.float64)
        comm.all_reduce(mm, "min")
        ok_range = float(mm[0]) == float(field.min()) and -float(mm[1]) == float(field.max())
        result_queue.put((rank, ok_carry, ok_halo, ok_sums, ok_range))
    finally:
        dist.destroy_process_group()


def test_sharded_host_logic_gloo_world2():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    results = [q.get(timeout=240) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, ok_carry, ok_halo, ok_sums, ok_range in results:
        assert ok_carry, f"rank {rank}: Lorenzo carry"
        assert ok_halo, f"rank {rank}: halo planes"
        assert ok_sums, f"rank {rank}: exact int128 combination"
        assert ok_range, f"rank {rank}: global value range"


def test_shard_planes_alignment():
    from paper_2603_25206_b200 import pipeline

    for n0, world in [(2048, 1), (2048, 2), (2048, 4), (2048, 8), (100, 3), (64, 4)]:
        bounds = [pipeline.shard_planes(n0, world, r, 16) for r in range(world)]
        assert bounds[0][0] == 0 and bounds[-1][1] == n0
        for (a, b), (c, _) in zip(bounds, bounds[1:]):
            assert b == c and a % 16 == 0 and b % 16 == 0
    with pytest.raises(ValueError):
        pipeline.shard_planes(16, 4, 0, 16)     # 16 planes cannot feed 4 ranks at 16-plane alignment


def test_finalize_matches_reference_expressions():
    from paper_2603_25206_b200 import pipeline

    rng = np.random.default_rng(3)
    q = rng.integers(-1000, 1000, size=5000).astype(np.int32)
    s1, s2 = O.exact_sum(q), O.exact_dot(q, q)
    mean, var = pipeline.finalize_mean_var(s1, s2, q.size, 0.01)
    assert mean == O.mean_from_dq(q, 0.01)
    assert var == O.var_from_dq(q, 0.01)
