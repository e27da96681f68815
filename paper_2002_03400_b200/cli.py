"""Drop-in command line for the GPU construction path.

Mirrors the reference CLI (tools/bfly_cli.cpp) for the subcommands on the
hot path:

  python -m paper_2002_03400_b200.cli [common options] factorize --config cfg.json
  python -m paper_2002_03400_b200.cli [common options] verify --config cfg.json [--check-eps e]
  python -m paper_2002_03400_b200.cli [common options] synth --levels L --rank r

Common options are the reference's (bfly_cli.cpp:345-354): --out, --csv,
--seed, --eps, --L, --r0, --oversample (--threads is accepted and ignored:
the GPU schedules itself).  ``factorize`` writes ``butterfly.bfh`` (reference
container format), ``log.json`` (log_to_json, bfly_cli.cpp:77-93) and, with
--csv, appends one ``bfly.factorize.v1`` row
(operator,n,L,eps,max_rank,error,seconds,bytes,matvec_columns; docs/formats.md
of the reference), exactly as run_factorize (bfly_cli.cpp:172-200).

Operator kinds in the config JSON ({"operator": kind, ...}):
  synthetic          the reference's seeded butterfly (real): levels, rank, seed
  nufft1d            config 0: n
  helmholtz_plates   config 1: n (a square)
  helmholtz_circle   config 2: n
  nufft_composition  config 3: n
  recompress         config 4: n
The Scattering2D / hemisphere Helmholtz kinds of the reference are outside
this path; reference operators can still be factorized
on the GPU from C++ through include/bfly_b200.hpp.
"""
from __future__ import annotations

import argparse
import json
import os
import sys

import numpy as np

from . import api, configs

KINDS = {"nufft1d": 0, "helmholtz_plates": 1, "helmholtz_circle": 2, "nufft_composition": 3, "recompress": 4}
SCHEMA = "bfly.factorize.v1"
HEADER = "operator,n,L,eps,max_rank,error,seconds,bytes,matvec_columns"


def fmt(v: float) -> str:
    """std::setprecision(17) formatting of the reference (bfly_cli.cpp:50-54)."""
    return f"{v:.17g}"


def append_csv(path: str, schema: str, header: str, rows):
    """bfly_cli.cpp:58-65: version comment + header when the file is new."""
    fresh = not os.path.exists(path)
    with open(path, "a") as f:
        if fresh:
            f.write(f"# schema: {schema}\n{header}\n")
        for r in rows:
            f.write(r + "\n")


def log_to_json(log: api.FactorizationLog) -> dict:
    """bfly_cli.cpp:77-93."""
    phases = [{"name": p.name, "forward_columns": p.forward_columns, "transpose_columns": p.transpose_columns,
               "seconds": p.seconds, "rounds": p.rounds, "probe_width": p.probe_width} for p in log.phases]
    return {"phases": phases, "forward_columns": log.forward_columns(),
            "transpose_columns": log.transpose_columns(), "total_columns": log.total_columns(),
            "peak_probe_bytes": log.peak_probe_bytes, "peak_concurrent_probes": log.peak_concurrent_probes,
            "rank_capped": bool(log.rank_capped), "total_seconds": log.total_seconds}


def build_operator(cfg: dict, opts) -> tuple:
    """-> (kind, op, row_tree, col_tree, levels, bytes per scalar)."""
    kind = cfg["operator"]
    seed = int(cfg.get("seed", opts.seed))
    if kind == "synthetic":
        levels = opts.L if opts.L > 0 else int(cfg.get("levels", 4))
        rank = int(cfg.get("rank", 8))
        bf = api.synth_butterfly(levels, rank, seed, scalar=api.REAL64)
        op = api.ButterflyOperator(bf)
        t = api.PartitionTree.build(np.arange(op.rows, dtype=float), levels)
        return kind, op, t, t, levels, 8
    if kind in KINDS:
        w = configs.build(KINDS[kind], int(cfg["n"]) if "n" in cfg else None,
                          levels=opts.L if opts.L > 0 else cfg.get("levels"))
        return kind, w.op, w.row_tree, w.col_tree, w.recon.levels, 16
    raise api.PreconditionError(f"unknown operator kind: {kind}")


def cmd_factorize(opts) -> int:
    if not opts.config:
        raise api.PreconditionError("factorize: --config is required")
    with open(opts.config) as f:
        cfg = json.load(f)
    kind, op, rt, ct, levels, scalar_bytes = build_operator(cfg, opts)
    rc = api.ReconstructionConfig(tolerance=opts.eps, rank_guess=opts.r0, oversampling=opts.oversample,
                                  levels=levels, seed=opts.seed)
    bf, log = api.factorize(op, rt, ct, rc)
    err = api.estimate_error(op, bf, 16, opts.seed)
    os.makedirs(opts.out, exist_ok=True)
    with open(os.path.join(opts.out, "butterfly.bfh"), "wb") as f:
        f.write(bf.serialize())
    with open(os.path.join(opts.out, "log.json"), "w") as f:
        f.write(json.dumps(log_to_json(log), indent=2) + "\n")
    if opts.csv:
        row = ",".join([kind, str(op.cols), str(levels), fmt(opts.eps), str(bf.max_rank()), fmt(err),
                        fmt(log.total_seconds), str(bf.nnz() * scalar_bytes), str(log.total_columns())])
        append_csv(opts.csv, SCHEMA, HEADER, [row])
    print(f"n={op.cols} L={levels} eps={opts.eps:g} max_rank={bf.max_rank()} error={err:g} "
          f"matvec_columns={log.total_columns()} nnz={bf.nnz()}")
    if log.rank_capped:
        print("warning: adaptive rank search hit the hard cap")
    return 0


def cmd_verify(opts) -> int:
    """run_verify (bfly_cli.cpp:203-235): factorize, then check the level-wise
    error bounds of Theorems 5.1-5.3 against a dense copy of the operator:
    column-basis sum at row level l <= (L - l + 1) e^2 ||K||^2 (l = L..l_m),
    row-basis sum <= (l + 1) e^2 ||K||^2 (l = 0..l_m), combined at l_m <=
    (L + 2) e^2 ||K||^2, e = --check-eps (default --eps).  Exit 0 iff all pass."""
    if not opts.config:
        raise api.PreconditionError("verify: --config is required")
    with open(opts.config) as f:
        cfg = json.load(f)
    kind, op, rt, ct, levels, _ = build_operator(cfg, opts)
    if op.rows * op.cols > opts.dense_cap * opts.dense_cap:
        raise api.PreconditionError("verify: operator exceeds the dense extraction cap")
    rc = api.ReconstructionConfig(tolerance=opts.eps, rank_guess=opts.r0, oversampling=opts.oversample,
                                  levels=levels, seed=opts.seed)
    bf, log = api.factorize(op, rt, ct, rc)
    res = api.residuals(op, bf)
    check_eps = opts.check_eps if opts.check_eps > 0 else opts.eps
    e2, kf2 = check_eps * check_eps, res["knorm2"]
    L, lm = bf.levels, bf.center
    ok = True

    def report(name, level, residual, bound):
        nonlocal ok
        passed = residual <= bound
        ok = ok and passed
        print(f"{name} level {level}: residual {residual:g} bound {bound:g}{'  pass' if passed else '  FAIL'}")

    for i, l in enumerate(range(L, lm - 1, -1)):
        report("column-basis bound", l, res["u"][i], (L - l + 1) * e2 * kf2)
    for l in range(0, lm + 1):
        report("row-basis bound", l, res["v"][l], (l + 1) * e2 * kf2)
    report("combined bound", lm, res["center"], (L + 2) * e2 * kf2)
    print(f"relative apply error: {api.estimate_error(op, bf, 16, opts.seed):g}")
    return 0 if ok else 1


def cmd_synth(opts) -> int:
    """bfly_cli.cpp:150-170: a ground-truth synthetic butterfly + manifest."""
    bf = api.synth_butterfly(opts.levels, opts.rank, opts.seed, scalar=api.REAL64)
    os.makedirs(opts.out, exist_ok=True)
    container = os.path.join(opts.out, "butterfly.bfh")
    with open(container, "wb") as f:
        f.write(bf.serialize())
    manifest = {"n": bf.rows, "levels": opts.levels, "rank": opts.rank, "seed": opts.seed, "scalar": "real64",
                "container": container, "nnz": bf.nnz()}
    with open(os.path.join(opts.out, "manifest.json"), "w") as f:
        f.write(json.dumps(manifest, indent=2) + "\n")
    print(f"wrote {container} (n={bf.rows}, L={opts.levels}, r={opts.rank})")
    return 0


def parser() -> argparse.ArgumentParser:
    ap = argparse.ArgumentParser(prog="bfly", description="B200 butterfly construction (drop-in CLI)")
    ap.add_argument("--config", default="", help="operator config JSON")
    ap.add_argument("--out", default=".", help="output directory")
    ap.add_argument("--csv", default="", help="CSV output path (appended)")
    ap.add_argument("--seed", type=int, default=0, help="random seed")
    ap.add_argument("--threads", type=int, default=1, help="accepted for compatibility; unused on the GPU")
    ap.add_argument("--eps", type=float, default=1e-3, help="truncation tolerance")
    ap.add_argument("--L", type=int, default=-1, help="tree depth override")
    ap.add_argument("--r0", type=int, default=4, help="initial rank guess")
    ap.add_argument("--oversample", type=int, default=2, help="oversampling columns")
    ap.add_argument("--dense-cap", dest="dense_cap", type=int, default=4096, help="dense-oracle size cap")
    sub = ap.add_subparsers(dest="cmd", required=True)
    f = sub.add_parser("factorize", help="reconstruct a butterfly from black-box products")
    f.add_argument("--config", dest="config_sub", default="")
    v = sub.add_parser("verify", help="check the level-wise error bounds densely")
    v.add_argument("--config", dest="config_sub", default="")
    v.add_argument("--check-eps", dest="check_eps", type=float, default=-1.0,
                   help="bound-evaluation tolerance (default: --eps)")
    s = sub.add_parser("synth", help="generate a ground-truth butterfly")
    s.add_argument("--levels", type=int, default=4)
    s.add_argument("--rank", type=int, default=4)
    return ap


def main(argv=None) -> int:
    opts = parser().parse_args(argv)
    if getattr(opts, "config_sub", ""):
        opts.config = opts.config_sub
    try:
        if opts.cmd == "factorize":
            return cmd_factorize(opts)
        if opts.cmd == "verify":
            return cmd_verify(opts)
        return cmd_synth(opts)
    except api.BflyError as e:  # the reference prints the error and exits non-zero
        print(f"error: {e}", file=sys.stderr)
        return 1


if __name__ == "__main__":
    sys.exit(main())
