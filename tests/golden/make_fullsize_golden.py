"""Full-size golden fixtures for the BASELINE configs.

Run ONCE on the GPU box's host cores (oracle/_ref travels there prebuilt; this
script needs no GPU and never touches the product library):

    python tests/golden/make_fullsize_golden.py --cfg 0 1 2 4 --out gpurun_out/golden

then copy gpurun_out/golden/full_cfg*.npz into tests/golden/.

Producers (both are test infrastructure):
  configs 0, 1, 2  the REFERENCE implementation itself (oracle/_ref/libbfly_ref.so:
                   /root/reference/proj/include/bfly compiled unmodified against
                   the Eigen-API shim) -- factorize() (reconstruct.hpp:412-419) at
                   the BASELINE size with cfg.threads = all host threads;
  config 4         the plain-C oracle (oracle/bo_*.c, pinned to the reference at
                   n <= 4096 by tests/test_ref_pin.py): the reference's own
                   ButterflyOperator runs its black box as single-threaded
                   Eigen-shim GEMMs (operators.hpp:105-122), ~16 TFLOP at n=262144,
                   far beyond any CPU budget; the oracle's apply is block-parallel.

Each full_cfg<k>.npz holds
  rank_profile      every block of every level (u levels lm..L, v levels 0..lm)
  phases            per phase (forward cols, transpose cols, rounds, probe width)
  phase_names, phase_seconds, total_seconds   the producer's FactorizationLog
  est_err           estimate_error(op, bf, 16, EST_SEED) (reconstruct.hpp:423-434)
  rows, yn_rows, yh_rows
                    sampled rows of bf.apply(X) and bf.apply_adjoint(Y) for the
                    seeded probes X = gaussian_matrix(n, 16, seed_mix(0, 5)),
                    Y = gaussian_matrix(n, 16, seed_mix(0, 6))
  yn_proj, yh_proj  G^H bf.apply(X), G^H bf.apply_adjoint(Y) with
                    G = gaussian_matrix(n, 8, seed_mix(0, 7)): random linear
                    functionals of EVERY output row, so the parity test covers the
                    whole output while the fixture stays small
  yn_colnorm, yh_colnorm  column norms of the full outputs
  threads, nproc, cpu_model, producer, wall_seconds
"""
import argparse
import os
import platform
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, os.path.join(ROOT, "oracle"))
sys.path.insert(0, os.path.join(ROOT, "tests"))

import oracle as O  # noqa: E402
from helpers import oracle_config  # noqa: E402

FULL_N = {0: 4096, 1: 16384, 2: 65536, 4: 262144}
EST_SEED = 3
N_ROWS = 512


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return platform.processor()


def probes(n):
    x = O.gaussian_matrix(n, 16, O.seed_mix(0, 5))
    y = O.gaussian_matrix(n, 16, O.seed_mix(0, 6))
    g = O.gaussian_matrix(n, 8, O.seed_mix(0, 7))
    rows = np.sort(np.random.default_rng(1234).choice(n, min(N_ROWS, n), replace=False))
    return x, y, g, rows


def summarize(yn, yh, g, rows):
    return dict(rows=rows, yn_rows=yn[rows], yh_rows=yh[rows], yn_proj=g.conj().T @ yn, yh_proj=g.conj().T @ yh,
                yn_colnorm=np.linalg.norm(yn, axis=0), yh_colnorm=np.linalg.norm(yh, axis=0))


def run_reference(cfg_id, n, threads):
    import refpy as R
    from test_ref_pin import _ref_config

    R.lib().ref_set_threads(threads)
    op, L, tol, r0 = _ref_config(cfg_id, n)
    t0 = time.perf_counter()
    bf = R.factorize(op, tol, r0, L, seed=0, threads=threads)
    wall = time.perf_counter() - t0
    phases, total = bf.log()
    ps = bf.phase_seconds()
    x, y, g, rows = probes(n)
    d = summarize(bf.apply(x, 0), bf.apply(y, 2), g, rows)
    d.update(rank_profile=bf.rank_profile(L).astype(np.int16), phases=np.array(phases, np.int64),
             phase_names=np.array([p[0] for p in ps]), phase_seconds=np.array([p[1] for p in ps]),
             total_seconds=total, est_err=bf.estimate_error(16, EST_SEED), wall_seconds=wall,
             producer="reference (oracle/_ref: reference headers + Eigen-API shim)")
    return d


def run_oracle(cfg_id, n, threads):
    O.set_threads(threads)
    op, rt, ct, cfg = oracle_config(cfg_id, n)
    t0 = time.perf_counter()
    bf, log = O.factorize(op, rt, ct, dict(cfg, threads=threads))
    wall = time.perf_counter() - t0
    x, y, g, rows = probes(n)
    d = summarize(bf.apply(x), bf.apply_adjoint(y), g, rows)
    ph = log["phases"]
    d.update(rank_profile=bf.rank_profile().astype(np.int16),
             phases=np.array([(p["forward_columns"], p["transpose_columns"], p["rounds"], p["probe_width"]) for p in ph],
                             np.int64),
             phase_names=np.array([p["name"] for p in ph]), phase_seconds=np.array([p["seconds"] for p in ph]),
             total_seconds=log["total_seconds"], est_err=O.estimate_error(op, bf, 16, EST_SEED), wall_seconds=wall,
             producer="C oracle (oracle/bo_*.c)")
    return d


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--cfg", type=int, nargs="+", default=[0, 1, 2, 4])
    ap.add_argument("--out", default=os.path.join(ROOT, "gpurun_out", "golden"))
    ap.add_argument("--threads", type=int, default=os.cpu_count() or 1)
    ap.add_argument("--n", type=int, default=0, help="override the size (smoke runs of this script)")
    a = ap.parse_args()
    os.makedirs(a.out, exist_ok=True)
    for c in a.cfg:
        n = a.n or FULL_N[c]
        run = run_oracle if c == 4 else run_reference
        d = run(c, n, a.threads)
        d.update(cfg=c, n=n, threads=a.threads, nproc=os.cpu_count(), cpu_model=cpu_model(), est_seed=EST_SEED)
        path = os.path.join(a.out, f"full_cfg{c}.npz" if not a.n else f"full_cfg{c}_n{n}.npz")
        np.savez_compressed(path, **d)
        print(f"cfg {c} n={n}: {d['producer']} total {float(d['total_seconds']):.1f} s (wall {d['wall_seconds']:.1f} s, "
              f"{a.threads} threads), max rank {int(d['rank_profile'].max())}, est_err {float(d['est_err']):.3e} -> {path}",
              flush=True)


if __name__ == "__main__":
    main()
