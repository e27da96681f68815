"""Times factorize() on the BASELINE configs (GPU) and prints the log."""
import argparse
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2002_03400_b200 as B  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--cfg", type=int, nargs="+", default=[0, 1, 2])
    ap.add_argument("--n", type=int, default=0)
    ap.add_argument("--reps", type=int, default=2)
    ap.add_argument("--profile", action="store_true")
    ap.add_argument("--c64", action="store_true", help="complex64 operators")
    a = ap.parse_args()
    for c in a.cfg:
        t0 = time.time()
        w = B.configs.build(c, a.n or None, scalar=B.COMPLEX64 if a.c64 else B.COMPLEX128)
        t1 = time.time()
        for r in range(a.reps):
            if a.profile and r == a.reps - 1:
                w.op.ctx.profile(-1)
                w.op.ctx.profile(1)
            bf, log = B.factorize(w.op, w.row_tree, w.col_tree, w.recon)
            if a.reps > 1:
                worst = max(log.phases, key=lambda p: p.seconds)
                print(f"   rep {r}: construct {log.total_seconds:.4f}s (slowest phase {worst.name} {worst.seconds*1e3:.1f} ms)")
        if a.profile:
            for k, v in sorted(w.op.ctx.profile_report().items(), key=lambda kv: -kv[1]["ms"]):
                print(f"   kernel {k:22s} launches {v['launches']:5d} ms {v['ms']:9.2f} "
                      f"TF/s {v['flops'] / max(v['ms'], 1e-9) / 1e9:7.2f} GB/s {v['bytes'] / max(v['ms'], 1e-9) / 1e6:8.1f}")
            w.op.ctx.profile(0)
        prof = bf.rank_profile()
        err = B.estimate_error(w.op, bf, 16, 0)
        print(f"cfg {c} {w.name}: setup {t1-t0:.2f}s construct {log.total_seconds:.4f}s "
              f"flops {log.flops/1e12:.3f} TF -> {log.flops/log.total_seconds/1e9:.1f} GFLOP/s, "
              f"evals {log.kernel_evals:.3e}, err {err:.2e}, nnz {bf.nnz()}, max rank {bf.max_rank()}")
        for p in log.phases:
            print(f"   {p.name:14s} {p.seconds*1e3:9.2f} ms fwd {p.forward_columns:6d} tr {p.transpose_columns:6d} "
                  f"rounds {p.rounds} width {p.probe_width}")
        print("   ranks per level (min/max):", [(int(r.min()), int(r.max())) for r in prof])
        sys.stdout.flush()


if __name__ == "__main__":
    main()
