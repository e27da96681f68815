"""Host-staged transport over torch.distributed (bfly_ctx_set_host_comm).

The library drains its stream, stages each exchange through pinned host
memory and calls these functions; here they run the matching
torch.distributed collectives on CPU tensors (gloo).  This is how several
processes that share ONE GPU run the real sharded construction and the
distributed apply (NCCL rejects two ranks on one device): every exchange is
a host round trip, no kernel ever waits on another rank.  On a multi-GPU
node the NCCL transport (Context.set_comm) is the product path.

The reference has no transport at all: its distributed layer is a
tally-only simulation (/root/reference/proj/include/bfly/layout.hpp:195-266).
"""
from __future__ import annotations

import ctypes as C
import traceback

import numpy as np

from ._native import HC_ALLGATHER, HC_ALLREDUCE, HC_SENDRECV, HostCommFns

_DT = {0: np.int32, 1: np.float64, 2: np.float32}


def _view(ptr, nbytes, dtype=np.uint8):
    if nbytes == 0:
        return np.zeros(0, dtype)
    buf = (C.c_uint8 * nbytes).from_address(ptr)
    return np.frombuffer(buf, dtype=dtype)


class TorchHostComm:
    """Collectives of one process group (default: the world group).  Keep the
    object alive as long as the context uses it (the Context does)."""

    def __init__(self, group=None):
        import torch.distributed as dist

        self.dist, self.group = dist, group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        self.calls = {"allgather": 0, "allreduce": 0, "sendrecv": 0}
        self.bytes = 0
        self._ag = HC_ALLGATHER(self._allgather)
        self._ar = HC_ALLREDUCE(self._allreduce)
        self._sr = HC_SENDRECV(self._sendrecv)
        self.fns = HostCommFns(None, self._ag, self._ar, self._sr)

    def _guard(self, fn, *a):
        try:
            fn(*a)
            return 0
        except Exception:  # the C side turns a nonzero code into BFLY_NCCL
            traceback.print_exc()
            return 1

    def _allgather(self, user, send, recv, nbytes):
        def run():
            import torch

            s = torch.from_numpy(_view(send, nbytes).copy())
            out = [torch.empty(nbytes, dtype=torch.uint8) for _ in range(self.world)]
            self.dist.all_gather(out, s, group=self.group)
            dst = _view(recv, nbytes * self.world)
            for r, t in enumerate(out):
                dst[r * nbytes:(r + 1) * nbytes] = t.numpy()
            self.calls["allgather"] += 1
            self.bytes += nbytes * self.world

        return self._guard(run)

    def _allreduce(self, user, buf, count, dtype, op):
        def run():
            import torch

            dt = _DT[dtype]
            v = _view(buf, count * np.dtype(dt).itemsize, dt)
            t = torch.from_numpy(v.copy())
            self.dist.all_reduce(t, op=self.dist.ReduceOp.MAX if op == 1 else self.dist.ReduceOp.SUM,
                                 group=self.group)
            v[:] = t.numpy()
            self.calls["allreduce"] += 1

        return self._guard(run)

    def _sendrecv(self, user, nsend, speer, sbuf, sbytes, nrecv, rpeer, rbuf, rbytes):
        def run():
            import torch

            reqs, recvs = [], []
            for i in range(nsend):
                t = torch.from_numpy(_view(sbuf[i], sbytes[i]).copy())
                reqs.append(self.dist.isend(t, int(speer[i]), group=self.group))
            for i in range(nrecv):
                t = torch.empty(int(rbytes[i]), dtype=torch.uint8)
                reqs.append(self.dist.irecv(t, int(rpeer[i]), group=self.group))
                recvs.append((i, t))
            for q in reqs:
                q.wait()
            for i, t in recvs:
                _view(rbuf[i], rbytes[i])[:] = t.numpy()
                self.bytes += int(rbytes[i])
            self.calls["sendrecv"] += 1

        return self._guard(run)
