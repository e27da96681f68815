"""Multi-rank host logic of the sharded construction, on CPU with gloo.

Two processes (world_size 2, gloo) each ask the product library (C ABI,
host-only entry points) which blocks they produce at every level, exchange
the lists over torch.distributed, and check the properties the device-side
exchange relies on: the per-rank lists partition every level exactly once,
leaf/W chunks are contiguous and start at rank * per_rank (the in-place
ncclAllGather layout), and R chunks are contiguous ranges of the nu-major
block order -- equal chunks at every level, so a level with fewer probes
than ranks splits a probe's partner nodes instead of idling ranks.  The same plan
drives tests/test_gpu_parity.py::test_virtual_ranks_match_single_gpu.
"""
import os
import socket

import pytest
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _plan(L, l, side, world, rank):
    import ctypes as C

    import numpy as np

    from paper_2002_03400_b200._native import lib

    n = lib().bfly_shard_blocks(L, l, side, world, rank, None)
    assert n >= 0
    out = np.zeros(max(n, 1), np.int64)
    lib().bfly_shard_blocks(L, l, side, world, rank, out.ctypes.data_as(C.c_void_p))
    return out[:n].tolist()


def _worker(rank, world, port, L, q):
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        errors = []
        nb = 1 << L
        cases = [(L, L, 0)] + [(L, l, 1) for l in range(1, L // 2 + 1)] + [(L, l, 2) for l in range(L // 2, L)]
        for (LL, l, side) in cases:
            mine = _plan(LL, l, side, world, rank)
            gathered = [None] * world
            dist.all_gather_object(gathered, mine)
            flat = [b for g in gathered for b in g]
            if sorted(flat) != list(range(nb)):
                errors.append(f"level {l} side {side}: not a partition")
            # every level: equal contiguous chunks of the 2^L blocks (levels with
            # fewer probes than ranks split a probe's partner nodes)
            per_rank = -(-nb // world)
            if side in (0, 1):
                for r, g in enumerate(gathered):
                    if g and (g != list(range(r * per_rank, r * per_rank + len(g)))):
                        errors.append(f"level {l} side {side} rank {r}: chunk not contiguous at r*per_rank")
            else:
                # nu-major order u = nu * 2^l + tau: contiguous unit ranges
                nnu, ntau = 1 << (L - l), 1 << l
                for r, g in enumerate(gathered):
                    units = [(b % nnu) * ntau + b // nnu for b in g]
                    if g and units != list(range(r * per_rank, r * per_rank + len(g))):
                        errors.append(f"level {l} rank {r}: R chunk is not a nu-major unit range")
            if max(len(g) for g in gathered) - min(len(g) for g in gathered) > per_rank:
                errors.append(f"level {l} side {side}: unbalanced chunks")
        # the all-gather itself: every rank ends with every rank's blocks
        import torch

        t = torch.tensor(_plan(L, L // 2, 2, world, rank), dtype=torch.int64)
        out = [torch.zeros_like(t) for _ in range(world)]
        dist.all_gather(out, t)
        if sorted(torch.cat(out).tolist()) != list(range(nb)):
            errors.append("tensor all_gather of the center level does not cover every block")
        q.put((rank, errors))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,L", [(2, 6), (2, 11)])
def test_shard_plan_two_ranks(world, L):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, L, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    for rank, errors in res:
        assert not errors, (rank, errors)


def test_shard_plan_edge_cases():
    """More ranks than probes: idle ranks own nothing; the union still covers."""
    for world in (3, 5, 8, 16):
        for L, l, side in ((4, 1, 1), (4, 3, 2), (3, 3, 0), (12, 6, 2)):
            lists = [_plan(L, l, side, world, r) for r in range(world)]
            flat = sorted(b for g in lists for b in g)
            assert flat == list(range(1 << L)), (world, L, l, side)
