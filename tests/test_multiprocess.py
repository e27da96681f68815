"""Multi-process path.

CPU (here): the host-staged transport's collectives over a world-size-2 gloo
group, and bench.py's self-launch (--gpus 2 spawns two ranks; a mismatched
WORLD_SIZE is refused).

GPU (one B200): the real sharded construction and the distributed apply run as
TWO PROCESSES on one GPU over the host-staged transport (tests/mp_worker.py
under torchrun): every rank ends with the same butterfly, equal to the
single-process factorization (identical rank profile of every block, apply
within 1e-12) and bit-identical to the same schedule executed in one process
(virtual_ranks = 2); every process layout's apply equals the plain apply.
"""
import json
import os
import socket
import subprocess
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


# ------------------------------------------------------------------ CPU
def _hc_worker(rank, world, port):
    import ctypes as C

    import torch.distributed as dist

    sys.path.insert(0, ROOT)
    from paper_2002_03400_b200.hostcomm import TorchHostComm

    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    hc = TorchHostComm()
    assert (hc.rank, hc.world) == (rank, world)
    # allgather: rank r contributes 5 bytes r*10 .. r*10+4
    send = np.arange(5, dtype=np.uint8) + 10 * rank
    recv = np.zeros(5 * world, np.uint8)
    assert hc.fns.allgather(None, send.ctypes.data, recv.ctypes.data, 5) == 0
    np.testing.assert_array_equal(recv, np.concatenate([np.arange(5, dtype=np.uint8) + 10 * r for r in range(world)]))
    # allreduce: int32 max, float64 sum, float32 sum
    a = np.array([rank, -rank, 7], np.int32)
    assert hc.fns.allreduce(None, a.ctypes.data, 3, 0, 1) == 0
    np.testing.assert_array_equal(a, [world - 1, 0, 7])
    d = np.array([0.5 + rank, 2.0])
    assert hc.fns.allreduce(None, d.ctypes.data, 2, 1, 0) == 0
    np.testing.assert_allclose(d, [0.5 * world + sum(range(world)), 2.0 * world])
    f = np.array([1.5], np.float32)
    assert hc.fns.allreduce(None, f.ctypes.data, 1, 2, 0) == 0
    assert f[0] == 1.5 * world
    # sendrecv: a ring, each rank sends (rank+1)*3 bytes to the next and receives from the previous
    nxt, prv = (rank + 1) % world, (rank - 1) % world
    sbuf = np.full((rank + 1) * 3, rank + 1, np.uint8)
    rbuf = np.zeros((prv + 1) * 3, np.uint8)
    i32, vp, i64 = C.c_int32, C.c_void_p, C.c_int64
    rc = hc.fns.sendrecv(None, 1, (i32 * 1)(nxt), (vp * 1)(sbuf.ctypes.data), (i64 * 1)(sbuf.size),
                         1, (i32 * 1)(prv), (vp * 1)(rbuf.ctypes.data), (i64 * 1)(rbuf.size))
    assert rc == 0
    np.testing.assert_array_equal(rbuf, np.full((prv + 1) * 3, prv + 1, np.uint8))
    # a failing collective reports a nonzero code (the library raises BFLY_NCCL)
    assert hc.fns.allreduce(None, a.ctypes.data, 3, 9, 0) != 0
    assert hc.calls == {"allgather": 1, "allreduce": 3, "sendrecv": 1}
    dist.destroy_process_group()


def _twice(fn):
    """A rendezvous port picked with bind(0) can be taken by another process
    before the ranks listen on it: one retry on a fresh port."""
    try:
        return fn()
    except Exception:  # noqa: BLE001
        return fn()


def test_host_comm_collectives_gloo_world2():
    import torch.multiprocessing as mp

    _twice(lambda: mp.spawn(_hc_worker, args=(2, _port()), nprocs=2, join=True))


def test_bench_self_launches_ranks():
    env = {k: v for k, v in os.environ.items() if k not in ("RANK", "WORLD_SIZE", "LOCAL_RANK")}

    def launch():
        r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--dry-launch"],
                           capture_output=True, text=True, timeout=300, env=env, cwd=ROOT)
        assert r.returncode == 0, r.stderr
        return r

    r = _twice(launch)
    lines = [json.loads(x) for x in r.stdout.splitlines() if x.startswith("{")]
    assert sorted((d["rank"], d["world"]) for d in lines) == [(0, 2), (1, 2)]
    assert "launching 2 ranks" in r.stderr


def test_bench_refuses_world_mismatch():
    env = dict(os.environ, RANK="0", WORLD_SIZE="3", LOCAL_RANK="0")
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--dry-launch"],
                       capture_output=True, text=True, timeout=120, env=env, cwd=ROOT)
    assert r.returncode == 2
    assert "refusing" in r.stderr


# ------------------------------------------------------------------ GPU
def _rel(a, b):
    return np.linalg.norm(a - b) / np.linalg.norm(b)


@pytest.mark.gpu
@pytest.mark.parametrize("cfg_id,n", [(2, 4096), (4, 16384), (3, 1024)])
def test_two_processes_one_gpu_host_transport(tmp_path, cfg_id, n):
    out = str(tmp_path / "mp")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2", "--master-addr",
           "127.0.0.1", "--master-port", str(_port()), os.path.join(ROOT, "tests", "mp_worker.py"),
           "--transport", "host", "--cfg", str(cfg_id), "--size", str(n), "--out", out]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=900, cwd=ROOT)
    print(r.stdout[-3000:], r.stderr[-3000:])
    assert r.returncode == 0
    assert "joined the host-staged communicator" in r.stderr
    ranks = [np.load(os.path.join(out, f"rank{i}.npz")) for i in range(2)]
    s = np.load(os.path.join(out, "single.npz"))
    for d in ranks:
        # the whole butterfly on every rank after the per-level all-gathers
        np.testing.assert_array_equal(d["profile"], s["profile"])
        np.testing.assert_array_equal(d["profile"], s["virt_profile"])
        assert _rel(d["yn"], s["yn"]) < 1e-12 and _rel(d["yh"], s["yh"]) < 1e-12
        # the same schedule in one process (virtual ranks): bit for bit
        np.testing.assert_array_equal(d["yn"], s["virt_yn"])
        np.testing.assert_array_equal(d["yh"], s["virt_yh"])
        assert abs(float(d["est"]) - float(s["est"])) < 1e-12
        # rounds and probe widths are the reference's on every rank
        np.testing.assert_array_equal(d["phases"][:, 2:], s["phases"][:, 2:])
        assert d["host_calls"][0] > 0  # level all-gathers went through the transport
        # distributed apply over the reference's process layouts (2 processes)
        for kind in ("column", "row", "hybrid"):
            assert _rel(d[f"layout_{kind}_n"], s["yn"]) < 1e-12
            assert _rel(d[f"layout_{kind}_h"], s["yh"]) < 1e-12
            # same exchange plan as the 2 virtual processes of the single run
            np.testing.assert_array_equal(d[f"layout_{kind}_moved"], s[f"layout_{kind}_moved"])
    np.testing.assert_array_equal(ranks[0]["yn"], ranks[1]["yn"])
    # transfer-phase black-box columns: the ranks' shares add up to the single run's
    tr = [i for i in range(len(s["phases"])) if i >= 2]
    tot = ranks[0]["phases"][tr, :2] + ranks[1]["phases"][tr, :2]
    np.testing.assert_array_equal(tot, s["phases"][tr, :2])
    # flops: the ranks' shares add up to the single-process construction's
    assert abs(float(ranks[0]["flops"]) + float(ranks[1]["flops"]) - float(s["flops"])) <= 1e-6 * float(s["flops"])
