#!/usr/bin/env python
"""Projected multi-GPU construction time from ONE GPU (a projection, not a
measurement): the factorization runs the sharded schedule for N virtual ranks
(virtual_ranks = N, every rank's share executed in turn on this GPU through
the same plan, pieces and exchange index math) with BFLY_VRANK_TIMING=1, which
records the device time of each rank's share of each phase.  Per phase

    projected = max over ranks of the share
              + (phase wall time - sum of the shares)   [work not split by rank:
                 leaf CPQR batches, rank read-backs, host planning -- kept whole]
              + all-gather of the phase's new blocks     [bytes / 700 GB/s + 30 us]

and the projected N-GPU time is the sum over phases.  Prints one JSON line per N.

  python tools/project_scaling.py [--cfg 2] [--ranks 2,4,8]
"""
import argparse
import ctypes as C
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ["BFLY_VRANK_TIMING"] = "1"

NVLINK_GBS = 700.0  # effective all-gather bus bandwidth assumed per GPU (NVLink 5: 900 GB/s per direction)
COLL_LAT_S = 30e-6


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--cfg", type=int, default=2)
    ap.add_argument("--n", type=int, default=0)
    ap.add_argument("--ranks", default="2,4,8")
    ap.add_argument("--reps", type=int, default=2)
    args = ap.parse_args()
    import dataclasses

    import numpy as np

    import paper_2002_03400_b200 as B
    from paper_2002_03400_b200._native import lib

    w = B.configs.build(args.cfg, args.n or None)
    for _ in range(args.reps):
        bf, log1 = B.factorize(w.op, w.row_tree, w.col_tree, w.recon)
    t1 = log1.total_seconds
    level_bytes = 16.0 * bf.nnz() / (len(log1.phases))  # mean factor bytes per phase (all-gather payload)
    out = {"cfg": args.cfg, "name": w.name, "one_gpu_s": round(t1, 4), "projection": []}
    for nr in [int(s) for s in args.ranks.split(",")]:
        rc = dataclasses.replace(w.recon, virtual_ranks=nr)
        for _ in range(args.reps):
            bf_n, log = B.factorize(w.op, w.row_tree, w.col_tree, rc)
        cnt = lib().bfly_vrank_times(None, 0)
        tab = np.zeros(max(cnt, 1))
        lib().bfly_vrank_times(tab.ctypes.data_as(C.c_void_p), cnt)
        tab = tab[:cnt].reshape(-1, nr) / 1e3  # seconds
        total, rows = 0.0, []
        for i, p in enumerate(log.phases):
            shares = tab[i] if i < len(tab) else np.zeros(nr)
            rest = max(0.0, p.seconds - shares.sum())
            gather = level_bytes * (nr - 1) / nr / (NVLINK_GBS * 1e9) + COLL_LAT_S
            t = shares.max() + rest + gather
            total += t
            rows.append({"phase": p.name, "max_share_ms": round(shares.max() * 1e3, 3),
                         "sum_shares_ms": round(shares.sum() * 1e3, 3), "unsplit_ms": round(rest * 1e3, 3),
                         "shares_ms": [round(float(x) * 1e3, 3) for x in shares]})
        out["projection"].append({"gpus": nr, "projected_s": round(total, 4), "speedup": round(t1 / total, 2),
                                  "phases": rows})
        print(json.dumps({"gpus": nr, "projected_s": round(total, 4), "speedup_vs_1gpu": round(t1 / total, 2)}),
              flush=True)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
