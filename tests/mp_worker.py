"""Worker of the multi-process tests (launched by torchrun; not collected by
pytest).  Every rank joins a torch.distributed group, binds a library
context to GPU (local_rank % device_count) and a transport:

  --transport host  the host-staged transport over gloo (bfly_ctx_set_host_comm):
                    runs with several ranks on ONE GPU -- every exchange is a host
                    round trip, no kernel waits on another rank;
  --transport nccl  the NCCL communicator (one GPU per rank).

It then runs the real sharded construction (factorizer.cu: probes and blocks
split across ranks, each level's new blocks all-gathered) and the distributed
apply over the reference's process layouts (dist.cu; layout.hpp:139-266), and
writes rank<r>.npz.  Rank 0 also writes single.npz: the same workload on a
fresh single-process context (no communicator), plain and with
virtual_ranks = world (the same schedule executed in one process).
"""
import argparse
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def probes(n, k, seed):
    rng = np.random.default_rng(seed)
    return np.asfortranarray(rng.standard_normal((n, k)) + 1j * rng.standard_normal((n, k)))


def run(B, ctx, a, world, virtual=0):
    import dataclasses

    w = B.configs.build(a.cfg, a.size, ctx=ctx)
    rc = dataclasses.replace(w.recon, virtual_ranks=virtual) if virtual else w.recon
    bf, log = B.factorize(w.op, w.row_tree, w.col_tree, rc)
    x = probes(w.op.cols, 4, 1)
    y = probes(w.op.rows, 4, 2)
    out = dict(profile=bf.rank_profile(), yn=bf.apply(x), yh=bf.apply_adjoint(y),
               phases=np.array([(p.forward_columns, p.transpose_columns, p.rounds, p.probe_width)
                                for p in log.phases], np.int64),
               flops=log.flops, est=B.estimate_error(w.op, bf, 16, 3))
    for kind in B.api.LAYOUT_KINDS:
        spec = B.api.LayoutSpec(kind, bf.levels, 8, world)
        yl, _, mv = bf.apply_layout(x, spec)
        xl, _, _ = bf.apply_layout(y, spec, trans=B.api.H)
        out[f"layout_{kind}_n"] = yl
        out[f"layout_{kind}_h"] = xl
        out[f"layout_{kind}_moved"] = np.array([mv["max_recv"], mv["total_recv"]])
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--cfg", type=int, default=2)
    ap.add_argument("--size", type=int, default=4096)
    ap.add_argument("--transport", default="host", choices=["host", "nccl"])
    ap.add_argument("--out", required=True)
    a = ap.parse_args()

    import torch
    import torch.distributed as dist

    import paper_2002_03400_b200 as B

    local = int(os.environ.get("LOCAL_RANK", 0))
    dev = local % torch.cuda.device_count()
    torch.cuda.set_device(dev)
    if a.transport == "host":
        dist.init_process_group("gloo")
    else:
        dist.init_process_group("nccl", device_id=torch.device("cuda", dev))
    rank, world = dist.get_rank(), dist.get_world_size()
    ctx = B.Context(dev)
    if a.transport == "host":
        hc = ctx.set_host_comm()
    else:
        uid = [B.Context.unique_id() if rank == 0 else None]
        dist.broadcast_object_list(uid, src=0)
        ctx.set_comm(rank, world, uid[0])
        hc = None
    info = ctx.comm_info()
    assert info == (rank, world, a.transport), info
    out = run(B, ctx, a, world)
    if hc is not None:
        out["host_calls"] = np.array([hc.calls["allgather"], hc.calls["allreduce"], hc.calls["sendrecv"]])
    os.makedirs(a.out, exist_ok=True)
    np.savez(os.path.join(a.out, f"rank{rank}.npz"), **out)
    dist.barrier()
    if rank == 0:
        c1 = B.Context(dev)
        single = run(B, c1, a, world)
        virt = run(B, c1, a, world, virtual=world)
        np.savez(os.path.join(a.out, "single.npz"), **single, **{f"virt_{k}": v for k, v in virt.items()})
    dist.barrier()
    dist.destroy_process_group()
    print(f"rank {rank}/{world} ok ({a.transport})", flush=True)


if __name__ == "__main__":
    main()
