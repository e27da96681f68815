"""Generates the golden fixtures in tests/golden/ from the REFERENCE itself.

Run here (where /root/reference exists and oracle/_ref is built):

    make -C oracle/ref ../_ref/libbfly_ref.so && python tests/golden/make_golden.py

Every expected value comes from oracle/_ref/libbfly_ref.so, i.e. the
reference's own headers (/root/reference/proj/include/bfly, unmodified)
compiled against the Eigen-API shim; only the input points are made by this
repository's seeded generators (the BASELINE workloads are builder-defined,
SURVEY.md App. A) and they are stored verbatim, so the fixtures do not depend
on the generators staying unchanged.

Files
  rng.npz      seed_mix (core.hpp:78-88) and gaussian_matrix (linalg.hpp:16-25)
               known answers, complex and real streams
  probe_kat.npz  first 64 Gaussians of every probe-seed family (leaf, W, R,
               error probe) of config 2
  cpqr.npz     pivoted_qr_truncate (linalg.hpp:63-80): ranks and bases
  layout.npz   process layouts (layout.hpp): comm_cost over a (kind, L, r, p)
               grid + rejected specs; assign_ownership maps and
               simulated_parallel_apply tallies on the reference's synthetic
               butterflies (L=4, 6; r=8, seed=L as acceptance criterion 6) and
               on the config-0 n=1024 factorization
  cfg_*.npz    factorize (reconstruct.hpp:412-419) on small BASELINE configs and
               the reference's synthetic butterfly: rank profile of every
               block, per-phase bookkeeping, butterfly apply / adjoint apply
               outputs on reference-generated probes, estimate_error, and the level-wise
               residual sums of the error-bound check (reconstruct.hpp:443-503)
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, os.path.join(ROOT, "oracle"))
sys.path.insert(0, os.path.join(ROOT, "tests"))

import oracle as O  # noqa: E402  (point generators + tree only)
import refpy as R  # noqa: E402
from helpers import _half_circle, _plate, _tree_order, _uniform  # noqa: E402

PROBE_COLS = 4

SEED_MIX_CASES = [(0,), (1,), (0xFFFFFFFFFFFFFFFF,), (42, 1), (42, 2), (7, 5), (7, 6), (123456789, 3, 4),
                  (2, 0x6d617472), (1, 2, 3, 4, 5)]


def make_rng():
    words = np.zeros((len(SEED_MIX_CASES), 5), np.uint64)
    nw = np.zeros(len(SEED_MIX_CASES), np.int32)
    out = np.zeros(len(SEED_MIX_CASES), np.uint64)
    for i, c in enumerate(SEED_MIX_CASES):
        words[i, : len(c)] = c
        nw[i] = len(c) - 1
        out[i] = R.seed_mix(c[0], *c[1:])
    d = dict(mix_words=words, mix_nwords=nw, mix_out=out)
    for tag, (rows, cols, seed) in dict(a=(7, 3, 42), b=(1, 1, 0), c=(257, 4, 2024), d=(5, 9, 123456789)).items():
        d[f"gz_{tag}"] = R.gaussian_matrix(rows, cols, seed, complex_=True)
        d[f"gz_{tag}_seed"] = np.uint64(seed)
        d[f"gd_{tag}"] = R.gaussian_matrix(rows, cols, seed, complex_=False)
    np.savez_compressed(os.path.join(HERE, "rng.npz"), **d)


def make_probe_kats():
    """First 64 Gaussians of every probe-seed family of config 2 (reconstruct.hpp
    seeds: leaf seed_mix(seed, tag, round) :370-372, W seed_mix(seed, 3, l, tau)
    :219, R seed_mix(seed, 4, l, nu) :275, error probe seed_mix(seed, 5) :428),
    drawn through gaussian_matrix (column-major fill, so any probe's first
    entries are these)."""
    seeds, words = [], []
    for tag in (1, 2):
        for rnd in range(3):
            words.append((0, tag, rnd))
    for l in (1, 3, 5):
        for node in (0, 1, (1 << l) - 1):
            words.append((0, 3, l, node))
            words.append((0, 4, l, node))
    words.append((0, 5))
    kat = np.zeros((len(words), 64), np.complex128)
    for i, w in enumerate(words):
        s = R.seed_mix(*w)
        seeds.append(s)
        kat[i] = R.gaussian_matrix(64, 1, s)[:, 0]
    wa = np.zeros((len(words), 4), np.uint64)
    nw = np.zeros(len(words), np.int32)
    for i, w in enumerate(words):
        wa[i, : len(w)] = w
        nw[i] = len(w)
    np.savez_compressed(os.path.join(HERE, "probe_kat.npz"), words=wa, nwords=nw, seeds=np.array(seeds, np.uint64),
                        first64=kat)


def make_cpqr():
    d = {}
    cases = []
    # rank-deficient + noise, full rank, exact rank 2 of 3, saturated wide, zero
    g = lambda r, c, s: R.gaussian_matrix(r, c, s, complex_=True)  # noqa: E731
    cases.append(("lowrank", g(40, 6, 1) @ g(6, 20, 2) + 1e-9 * g(40, 20, 3), 1e-6))
    cases.append(("full", g(16, 10, 4), 1e-6))
    a = g(64, 3, 5)
    a[:, 2] = a[:, 0] - 2.0j * a[:, 1]
    cases.append(("exact2", a, 1e-10))
    s = np.logspace(0, -12, 18)
    cases.append(("graded", (g(30, 18, 6) * s) @ g(18, 24, 7), 0.25e-6))
    cases.append(("wide", g(8, 20, 8), 1e-6))
    cases.append(("zero", np.zeros((5, 3), complex), 1e-8))
    for name, w, eps in cases:
        rank, q = R.pivoted_qr_truncate(w, eps)
        d[f"{name}_w"] = w
        d[f"{name}_eps"] = eps
        d[f"{name}_rank"] = rank
        d[f"{name}_q"] = q
    d["names"] = np.array([c[0] for c in cases])
    np.savez_compressed(os.path.join(HERE, "cpqr.npz"), **d)


def config_inputs(cfg_id, n):
    """-> dict of stored inputs + the reference operator"""
    L = O.depth_for(n, 32)
    if cfg_id == 0:
        x, _ = _tree_order(_uniform(n, 0, 1, 0.0, 1.0), L, 1)
        xi, _ = _tree_order(_uniform(n, 0, 2, -n / 2.0, n / 2.0), L, 1)
        inp = dict(kind=1, rows_pts=x, cols_pts=xi, kappa=0.0, dim=1, L=L, tol=1e-6, r0=16)
    elif cfg_id == 1:
        side = int(round(np.sqrt(n)))
        t, _ = _tree_order(_plate(side, 0.0), L, 3)
        s, _ = _tree_order(_plate(side, 2.0), L, 3)
        inp = dict(kind=2, rows_pts=t, cols_pts=s, kappa=2.0 * np.pi / (10.0 * (1.0 / side)), dim=3, L=L, tol=1e-6,
                   r0=16)
    elif cfg_id == 2:
        t, _ = _tree_order(_half_circle(n, True), L, 2)
        s, _ = _tree_order(_half_circle(n, False), L, 2)
        inp = dict(kind=3, rows_pts=t, cols_pts=s, kappa=2.0 * n / 10.0, dim=2, L=L, tol=1e-6, r0=4)
    elif cfg_id == 3:
        x1, xi1 = _uniform(n, 1, 1, 0.0, 1.0), _uniform(n, 1, 2, -n / 2.0, n / 2.0)
        x2, xi2 = _uniform(n, 2, 1, 0.0, 1.0), _uniform(n, 2, 2, -n / 2.0, n / 2.0)
        x2, _ = _tree_order(x2, L, 1)
        xi1, _ = _tree_order(xi1, L, 1)
        inp = dict(kind=4, rows_pts=x2, cols_pts=xi1, f2_cols=xi2, f1_rows=x1, kappa=0.0, dim=1, L=L, tol=1e-5, r0=16)
    else:
        raise ValueError(cfg_id)
    if cfg_id == 3:
        op = R.compose_op(n, inp["rows_pts"], inp["f2_cols"], inp["f1_rows"], inp["cols_pts"], L)
    else:
        op = R.kernel_op(inp["kind"], inp["rows_pts"], inp["cols_pts"], inp["kappa"], inp["dim"], L)
    return inp, op


def save_factorization(name, inp, op, bf, L, seed):
    rows, cols = op.rows, op.cols
    phases, _ = bf.log()
    x = R.gaussian_matrix(cols, PROBE_COLS, R.seed_mix(7, 5))
    y = R.gaussian_matrix(rows, PROBE_COLS, R.seed_mix(7, 6))
    d = dict(inp)
    d.update(seed=seed, rank_profile=bf.rank_profile(L), phases=np.array(phases, np.int64),
             probe_x=x, probe_y=y, apply_n=bf.apply(np.asfortranarray(x), 0),
             apply_h=bf.apply(np.asfortranarray(y), 2), estimate_error=bf.estimate_error(16, 3))
    u, v, cen, kn = bf.residuals(L, L // 2)
    d.update(res_u=u, res_v=v, res_center=cen, res_knorm2=kn)
    np.savez_compressed(os.path.join(HERE, f"{name}.npz"), **d)
    print(name, "ranks", int(d["rank_profile"].max()), "phases", len(phases))


def make_configs():
    for cfg_id, n in ((0, 1024), (1, 1024), (2, 1024), (3, 512)):
        inp, op = config_inputs(cfg_id, n)
        bf = R.factorize(op, inp["tol"], inp["r0"], inp["L"], seed=0, threads=8)
        save_factorization(f"cfg{cfg_id}_n{n}", inp, op, bf, inp["L"], 0)
    # the reference's own synthetic butterfly (operators.hpp:131-178) as the black box
    for L, r, seed in ((5, 4, 7), (4, 3, 21)):
        op = R.synth_op(L, r, seed)
        bf = R.factorize(op, 1e-10, 4, L, seed=seed + 1000)
        inp = dict(kind=0, L=L, rank=r, synth_seed=seed, tol=1e-10, r0=4)
        save_factorization(f"synth_L{L}_r{r}_s{seed}", inp, op, bf, L, seed + 1000)


def make_layout():
    d = {}
    grid, vals, bad = [], [], []
    for kind in (0, 1, 2):
        for L in range(1, 7):
            for r in (1, 2, 8):
                for p in [1 << g for g in range(L + 1)] + [3, 1 << (L + 1)]:
                    try:
                        v = R.comm_cost(kind, L, r, p)
                    except RuntimeError:
                        bad.append((kind, L, r, p))
                        continue
                    grid.append((kind, L, r, p))
                    vals.append(v)
    d["cc_spec"] = np.array(grid, np.int64)
    d["cc_val"] = np.array(vals)
    d["cc_bad"] = np.array(bad, np.int64)
    for L in (4, 6):
        specs, tall, own = [], [], []
        for kind in (0, 1, 2):
            for g in range(L + 1):
                t, o = R.layout_synth(L, 8, L, kind, 1 << g)
                specs.append((kind, 1 << g))
                tall.append(t)
                own.append(o)
        d[f"synth{L}_spec"] = np.array(specs, np.int64)
        d[f"synth{L}_tally"] = np.array(tall)
        d[f"synth{L}_owners"] = np.array(own, np.int32)
    inp, op = config_inputs(0, 1024)
    bf = R.factorize(op, inp["tol"], inp["r0"], inp["L"], seed=0, threads=8)
    specs, tall, own = [], [], []
    for kind in (0, 1, 2):
        for g in range(inp["L"] + 1):
            t, o = bf.layout(inp["L"], kind, 1 << g)
            specs.append((kind, 1 << g))
            tall.append(t)
            own.append(o)
    d["cfg0_spec"] = np.array(specs, np.int64)
    d["cfg0_tally"] = np.array(tall)
    d["cfg0_owners"] = np.array(own, np.int32)
    d["cfg0_L"] = inp["L"]
    np.savez_compressed(os.path.join(HERE, "layout.npz"), **d)
    print("layout", len(grid), "comm_cost cells,", len(bad), "rejected")


if __name__ == "__main__":
    assert R.available(), "build oracle/_ref first (make -C oracle/ref)"
    make_rng()
    make_probe_kats()
    make_cpqr()
    make_configs()
    make_layout()
