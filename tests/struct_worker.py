"""Worker of test_structured_butterfly_products (not collected by pytest).

Recompresses a butterfly operator over its own trees and writes the result.
The parent runs it with BFLY_NO_STRUCT_APPLY (the reference's padded products,
reconstruct.hpp:72-85), with BFLY_NO_LEAF_FUSE (structured products:
DevButterfly::apply_structured skips the blocks the probes' zero rows cannot
reach) and with neither (structured, the chain's leaf projection fused into
the black box's last stage), on the same seeds.
"""
import argparse
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--case", required=True)
    ap.add_argument("--out", required=True)
    ap.add_argument("--vr", type=int, default=0)
    a = ap.parse_args()
    import dataclasses

    import paper_2002_03400_b200 as B

    if a.case == "cfg4":
        w = B.configs.build(4, 4096)
        op, rt, ct, rc = w.op, w.row_tree, w.col_tree, w.recon
    elif a.case == "cfg4_c64":
        w = B.configs.build(4, 4096, scalar=B.COMPLEX64)
        op, rt, ct, rc = w.op, w.row_tree, w.col_tree, w.recon
    elif a.case == "synth_real":
        bf0 = B.synth_butterfly(6, 4, 9, scalar=B.REAL64)
        n = (1 << 6) * 8
        op = B.ButterflyOperator(bf0)
        rt = ct = B.PartitionTree.build(np.arange(n, dtype=float), 6)
        rc = B.ReconstructionConfig(levels=6, tolerance=1e-10, rank_guess=4, oversampling=2, seed=77)
    elif a.case == "ragged":
        # a butterfly with ragged leaves and varying ranks: the factorization of
        # config 2 at n = 1500, recompressed over the same trees
        w = B.configs.build(2, 1500)
        bf0, _ = B.factorize(w.op, w.row_tree, w.col_tree, w.recon)
        op = B.ButterflyOperator(bf0)
        rt, ct = w.row_tree, w.col_tree
        rc = dataclasses.replace(w.recon, tolerance=1e-8, seed=5)
    else:
        raise SystemExit(f"unknown case {a.case}")
    if a.vr:
        rc = dataclasses.replace(rc, virtual_ranks=a.vr)
    bf, log = B.factorize(op, rt, ct, rc)
    rng = np.random.default_rng(3)
    x = np.asfortranarray(rng.standard_normal((op.cols, 5)) + 1j * rng.standard_normal((op.cols, 5)))
    y = np.asfortranarray(rng.standard_normal((op.rows, 5)) + 1j * rng.standard_normal((op.rows, 5)))
    if a.case == "synth_real":
        x, y = np.asfortranarray(x.real), np.asfortranarray(y.real)
    if a.case == "cfg4_c64":
        x, y = x.astype(np.complex64), y.astype(np.complex64)
    np.savez(a.out, profile=bf.rank_profile(), yn=bf.apply(x), yh=bf.apply_adjoint(y), flops=log.flops,
             cols=np.array([(p.forward_columns, p.transpose_columns, p.rounds, p.probe_width) for p in log.phases]),
             seconds=log.total_seconds, struct=os.environ.get("BFLY_NO_STRUCT_APPLY") is None)


if __name__ == "__main__":
    main()
