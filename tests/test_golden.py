"""Golden fixtures (tests/golden/*.npz, made by tests/golden/make_golden.py
from the REFERENCE implementation itself, oracle/_ref).

CPU part: the C oracle reproduces every golden vector -- bit-exact for the
integer / RNG streams, identical ranks and bookkeeping for the
factorizations, apply outputs within round-off.  GPU part (-m gpu): the
sm_100a library reproduces the same vectors through its public API.  Nothing
here reads /root/reference: the fixtures are committed.
"""
import glob
import os

import numpy as np
import pytest

import oracle as O
from helpers import rel_err

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
CFG_FILES = sorted(glob.glob(os.path.join(GOLDEN, "cfg*.npz")) + glob.glob(os.path.join(GOLDEN, "synth*.npz")))
APPLY_TOL = 1e-10


def _load(name):
    return np.load(os.path.join(GOLDEN, name), allow_pickle=False)


def _mix_cases(g):
    for words, nw, out in zip(g["mix_words"], g["mix_nwords"], g["mix_out"]):
        yield int(words[0]), [int(w) for w in words[1 : 1 + nw]], int(out)


def _phase_tuples(log_phases):
    return [tuple(p) for p in log_phases]


# ------------------------------------------------------------------ oracle --
def test_oracle_seed_mix_golden():
    g = _load("rng.npz")
    for seed, words, out in _mix_cases(g):
        assert O.seed_mix(seed, *words) == out, (seed, words)


@pytest.mark.parametrize("tag", ["a", "b", "c", "d"])
def test_oracle_gaussian_golden_bit_exact(tag):
    g = _load("rng.npz")
    gz, gd = g[f"gz_{tag}"], g[f"gd_{tag}"]
    seed = int(g[f"gz_{tag}_seed"])
    rows, cols = gz.shape
    np.testing.assert_array_equal(O.gaussian_matrix(rows, cols, seed), gz)
    np.testing.assert_array_equal(O.gaussian_matrix(rows, cols, seed, real=True), gd)


def _probe_kats():
    g = _load("probe_kat.npz")
    for words, nw, seed, first in zip(g["words"], g["nwords"], g["seeds"], g["first64"]):
        yield [int(x) for x in words[:nw]], int(seed), first


def test_oracle_probe_seed_kats_bit_exact():
    """Every probe-seed family (leaf, W, R, error probe): the seed and the
    first 64 Gaussians of the probe equal the reference's bit for bit."""
    for words, seed, first in _probe_kats():
        assert O.seed_mix(*words) == seed, words
        np.testing.assert_array_equal(O.gaussian_matrix(64, 1, seed)[:, 0], first)


def test_oracle_cpqr_golden():
    g = _load("cpqr.npz")
    for name in g["names"]:
        w, eps, rank, q = g[f"{name}_w"], float(g[f"{name}_eps"]), int(g[f"{name}_rank"]), g[f"{name}_q"]
        qo, k, _, _ = O.pivoted_qr_truncate(w, eps)
        assert k == max(rank, 0), name
        if k:
            # trailing columns of the graded case sit at R_kk ~ 1e-7 |R_00|:
            # round-off is amplified there (same span, conditioning-limited)
            assert rel_err(qo, q) < (1e-9 if name == "graded" else 1e-12), name


def _oracle_problem(d):
    kind, L = int(d["kind"]), int(d["L"])
    if kind == 0:
        bf = O.synth_butterfly(L, int(d["rank"]), int(d["synth_seed"]))
        n = (1 << L) * 8
        t = O.PartitionTree.build(np.arange(n, dtype=float), L)
        return O.butterfly_operator(bf), t, t
    dim = int(d["dim"])
    rp, cp = d["rows_pts"], d["cols_pts"]
    rt = O.PartitionTree.build(rp[:, :dim], L, dim)
    ct = O.PartitionTree.build(cp[:, :dim], L, dim)
    assert (rt.perm == np.arange(len(rp))).all() and (ct.perm == np.arange(len(cp))).all()
    if kind == 4:
        f2 = O.kernel_operator(O.OP_NUFFT, rp, d["f2_cols"])
        f1 = O.kernel_operator(O.OP_NUFFT, d["f1_rows"], cp)
        return O.compose_operator(f2, f1), rt, ct
    okind = {1: O.OP_NUFFT, 2: O.OP_PLATES, 3: O.OP_CIRCLE}[kind]
    return O.kernel_operator(okind, rp, cp, float(d["kappa"])), rt, ct


@pytest.mark.parametrize("path", CFG_FILES, ids=[os.path.basename(p)[:-4] for p in CFG_FILES])
def test_oracle_factorization_golden(path, oracle_threads):
    d = np.load(path)
    op, rt, ct = _oracle_problem(d)
    cfg = dict(levels=int(d["L"]), tolerance=float(d["tol"]), rank_guess=int(d["r0"]), oversampling=2,
               seed=int(d["seed"]), threads=oracle_threads)
    bf, log = O.factorize(op, rt, ct, cfg)
    np.testing.assert_array_equal(bf.rank_profile(), d["rank_profile"])
    got = [(p["forward_columns"], p["transpose_columns"], p["rounds"], p["probe_width"]) for p in log["phases"]]
    assert got == _phase_tuples(d["phases"])
    assert rel_err(bf.apply(d["probe_x"]), d["apply_n"]) < APPLY_TOL
    assert rel_err(bf.apply_adjoint(d["probe_y"]), d["apply_h"]) < APPLY_TOL
    est = O.estimate_error(op, bf, 16, 3)
    assert abs(est - float(d["estimate_error"])) <= 1e-5 * float(d["estimate_error"]) + 1e-14


# --------------------------------------------------------------------- GPU --
@pytest.fixture(scope="module")
def B():
    import paper_2002_03400_b200 as B

    return B


@pytest.mark.gpu
def test_gpu_rng_golden(B):
    g = _load("rng.npz")
    for seed, words, out in _mix_cases(g):
        assert B.seed_mix(seed, *words) == out
    for tag in "abcd":
        gz, gd = g[f"gz_{tag}"], g[f"gd_{tag}"]
        seed = int(g[f"gz_{tag}_seed"])
        rows, cols = gz.shape
        # device log/sincos vs glibc: a few ulp (the stream itself is exact)
        assert np.max(np.abs(B.gaussian_matrix(rows, cols, seed) - gz)) <= 4e-15 * max(1.0, np.abs(gz).max())
        assert np.max(np.abs(B.gaussian_matrix(rows, cols, seed, scalar=B.REAL64) - gd)) <= 4e-15 * max(
            1.0, np.abs(gd).max())


@pytest.mark.gpu
def test_gpu_probe_seed_kats(B):
    for words, seed, first in _probe_kats():
        assert B.seed_mix(*words) == seed
        g = B.gaussian_matrix(64, 1, seed)[:, 0]
        assert np.max(np.abs(g - first)) <= 4e-15 * max(1.0, np.abs(first).max())


@pytest.mark.gpu
def test_gpu_cpqr_golden(B):
    g = _load("cpqr.npz")
    for name in g["names"]:
        w, eps, rank, q = g[f"{name}_w"], float(g[f"{name}_eps"]), int(g[f"{name}_rank"]), g[f"{name}_q"]
        qg = B.pivoted_qr_truncate(w, eps)
        assert qg.shape[1] == max(rank, 0), name
        if rank > 0:
            assert rel_err(qg, q) < 1e-10, name


def _gpu_problem(B, d):
    kind, L = int(d["kind"]), int(d["L"])
    if kind == 0:
        bf = B.synth_butterfly(L, int(d["rank"]), int(d["synth_seed"]))
        n = (1 << L) * 8
        t = B.PartitionTree.build(np.arange(n, dtype=float), L)
        return B.ButterflyOperator(bf), t, t
    dim = int(d["dim"])
    rp, cp = d["rows_pts"], d["cols_pts"]
    rt = B.PartitionTree.build(rp[:, :dim], L, dim)
    ct = B.PartitionTree.build(cp[:, :dim], L, dim)
    if kind == 4:
        f2 = B.NufftOperator(rp, d["f2_cols"])
        f1 = B.NufftOperator(d["f1_rows"], cp)
        return B.CompositionOperator(f2, f1), rt, ct
    if kind == 1:
        return B.NufftOperator(rp, cp), rt, ct
    if kind == 2:
        return B.HelmholtzPlatesOperator(rp, cp, float(d["kappa"])), rt, ct
    return B.HelmholtzCircleOperator(rp, cp, float(d["kappa"])), rt, ct


@pytest.mark.gpu
@pytest.mark.parametrize("path", CFG_FILES, ids=[os.path.basename(p)[:-4] for p in CFG_FILES])
def test_gpu_factorization_golden(B, path):
    d = np.load(path)
    op, rt, ct = _gpu_problem(B, d)
    rc = B.ReconstructionConfig(tolerance=float(d["tol"]), rank_guess=int(d["r0"]), levels=int(d["L"]),
                                seed=int(d["seed"]))
    bf, log = B.factorize(op, rt, ct, rc)
    np.testing.assert_array_equal(bf.rank_profile(), d["rank_profile"])
    got = [(p.forward_columns, p.transpose_columns, p.rounds, p.probe_width) for p in log.phases]
    assert got == _phase_tuples(d["phases"])
    assert rel_err(bf.apply(d["probe_x"]), d["apply_n"]) < APPLY_TOL
    assert rel_err(bf.apply_adjoint(d["probe_y"]), d["apply_h"]) < APPLY_TOL
    for k in (1, 2):  # narrow column counts take the per-stage kernel with several blocks per CTA
        assert rel_err(bf.apply(d["probe_x"][:, :k]), d["apply_n"][:, :k]) < APPLY_TOL
        assert rel_err(bf.apply_adjoint(d["probe_y"][:, :k]), d["apply_h"][:, :k]) < APPLY_TOL
    est = B.estimate_error(op, bf, 16, 3)
    assert abs(est - float(d["estimate_error"])) <= 1e-5 * float(d["estimate_error"]) + 1e-14


@pytest.mark.gpu
@pytest.mark.parametrize("path", CFG_FILES, ids=[os.path.basename(p)[:-4] for p in CFG_FILES])
def test_gpu_residual_sums_match_reference(B, path):
    """Level-wise residual sums of the error-bound check (reconstruct.hpp:
    443-503), computed on the GPU against its own dense copy of the operator,
    equal the reference's on its factorization of the same problem (identical
    ranks; the residuals are truncation-dominated, round-off far below)."""
    d = np.load(path)
    op, rt, ct = _gpu_problem(B, d)
    rc = B.ReconstructionConfig(tolerance=float(d["tol"]), rank_guess=int(d["r0"]), levels=int(d["L"]),
                                seed=int(d["seed"]))
    bf, _ = B.factorize(op, rt, ct, rc)
    r = B.residuals(op, bf)
    kn = float(d["res_knorm2"])
    assert abs(r["knorm2"] - kn) <= 1e-12 * kn
    floor = 1e-20 * kn  # exact recoveries: residuals at round-off
    np.testing.assert_allclose(r["u"], d["res_u"], rtol=1e-3, atol=floor)
    np.testing.assert_allclose(r["v"], d["res_v"], rtol=1e-3, atol=floor)
    assert abs(r["center"] - float(d["res_center"])) <= 1e-3 * float(d["res_center"]) + floor

