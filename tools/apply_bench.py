#!/usr/bin/env python
"""Butterfly apply timing on the config-2 factorization (n = 65536, L = 11):
device-resident x/y, L2 flushed before every call, CUDA events on the library
stream.  Prints one JSON line per k.  Knobs are the library's environment
variables (BFLY_APPLY_PERSIST, BFLY_PERSIST_DEPTH, BFLY_PERSIST_WPC, ...).

  python tools/apply_bench.py [--ks 1,2,16] [--reps 20] [--trans 0]
"""
import argparse
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--ks", default="1,2,16")
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--trans", type=int, default=0)
    ap.add_argument("--cfg", type=int, default=2)
    ap.add_argument("--synth", action="store_true", help="config 4's input butterfly (n=262144, leaf 64, rank 32)")
    args = ap.parse_args()
    import torch

    import paper_2002_03400_b200 as B

    if args.synth:
        ctx = B.Context(0)
        bf = B.synth_butterfly(12, 32, 0, leaf=64, perturb=1e-8, ctx=ctx)
    else:
        w = B.configs.build(args.cfg)
        bf, _ = B.factorize(w.op, w.row_tree, w.col_tree, w.recon)
        ctx = w.op.ctx
    stream = torch.cuda.ExternalStream(ctx.stream)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    lib, C = B.api.lib(), B.api.C
    nin, nout = (bf.cols, bf.rows) if args.trans == 0 else (bf.rows, bf.cols)
    for k in [int(s) for s in args.ks.split(",")]:
        x = torch.randn((k, nin), dtype=torch.complex128, device="cuda").t()
        y = torch.empty((k, nout), dtype=torch.complex128, device="cuda").t()

        def call():
            B.api.check(lib.bfly_apply(bf.h, args.trans, C.c_void_p(x.data_ptr()), nin, C.c_void_p(y.data_ptr()),
                                       nout, k, 1))

        for _ in range(3):
            call()
        torch.cuda.synchronize()
        ts = []
        for _ in range(args.reps):
            flush.zero_()
            torch.cuda.synchronize()
            a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a0.record(stream)
            call()
            a1.record(stream)
            a1.synchronize()
            ts.append(a0.elapsed_time(a1))
        ms = statistics.median(ts)
        nbytes = 16.0 * (bf.nnz() + (bf.rows + bf.cols) * k)
        print(json.dumps({"k": k, "trans": args.trans, "ms": round(ms, 4), "min_ms": round(min(ts), 4),
                          "GB/s": round(nbytes / ms / 1e6, 1), "frac_of_hbm": round(nbytes / ms / 1e6 / 6554.9, 3),
                          "persist": os.environ.get("BFLY_APPLY_PERSIST", "1")}), flush=True)


if __name__ == "__main__":
    main()
