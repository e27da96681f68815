"""CPU oracle checked against the reference's own test expectations.

The reference pins properties, not values: these are its
Catch2 cases (tests/test_linalg.cpp, test_reconstruct.cpp,
test_butterfly.cpp) restated against the oracle, so the checker the GPU
parity tests rely on is itself pinned to the reference's behaviour.
"""
import numpy as np
import pytest

import oracle as O
from helpers import oracle_config, rel_err


def exact_rank(m, n, r, seed, real=True):
    left = O.gaussian_matrix(m, r, seed, real=real)
    right = O.gaussian_matrix(r, n, seed + 1, real=real)
    q = O.householder_q(left)
    return q @ right


# ---------------------------------------------------------------- linalg
def test_gaussian_deterministic_and_seed_sensitive():
    """test_linalg.cpp:30-45"""
    assert np.array_equal(O.gaussian_matrix(3, 2, 7, real=True), O.gaussian_matrix(3, 2, 7, real=True))
    assert np.abs(O.gaussian_matrix(4, 4, 1, True) - O.gaussian_matrix(4, 4, 2, True)).max() > 0
    assert np.array_equal(O.gaussian_matrix(3, 3, 11), O.gaussian_matrix(3, 3, 11))
    with pytest.raises(O.OracleError):
        O.gaussian_matrix(0, 2, 1)


def test_gaussian_moments():
    """test_linalg.cpp:47-52"""
    g = O.gaussian_matrix(2048, 1, 42, real=True)
    assert abs(g.mean()) < 0.1
    assert abs(g.var(ddof=1) - 1.0) < 0.15


def test_cpqr_identity_and_rank_one():
    """test_linalg.cpp:54-68"""
    q, k, _, _ = O.pivoted_qr_truncate(np.eye(4), 1e-6)
    assert k == 4
    assert np.linalg.norm(q.conj().T @ q - np.eye(4)) < 2e-12
    u = O.gaussian_matrix(8, 1, 3, True)[:, 0]
    v = O.gaussian_matrix(8, 1, 4, True)[:, 0]
    u /= np.linalg.norm(u)
    v /= np.linalg.norm(v)
    w = np.outer(u, v)
    q, k, _, _ = O.pivoted_qr_truncate(w, 1e-10)
    assert k == 1
    assert np.linalg.norm(w - q @ (q.conj().T @ w)) <= 1e-12 * np.linalg.norm(w)


def test_cpqr_tracks_svd_oracle():
    """test_linalg.cpp:70-88"""
    w = O.gaussian_matrix(16, 16, 9, True).real
    u, _, vt = np.linalg.svd(w)
    sv = 10.0 ** (-0.5 * np.arange(16))
    w = (u * sv) @ vt
    eps = 1e-3
    q, k, _, _ = O.pivoted_qr_truncate(w, eps)
    resid = np.linalg.norm(w - q @ (q.conj().T @ w))
    oracle = np.sqrt(np.sum(sv[sv <= eps * sv[0]] ** 2))
    assert resid <= 4 * eps * np.linalg.norm(w)
    assert resid <= 10 * max(oracle, 1e-15 * np.linalg.norm(w)) + eps * np.linalg.norm(w)


def test_cpqr_zero_and_idempotent():
    """test_linalg.cpp:90-103"""
    q, k, _, _ = O.pivoted_qr_truncate(np.zeros((5, 3)), 1e-8)
    assert k == 0
    w = O.gaussian_matrix(12, 5, 17, True)
    q1, k1, _, _ = O.pivoted_qr_truncate(w, 1e-10)
    q2, k2, _, _ = O.pivoted_qr_truncate(q1, 1e-10)
    assert k1 == k2
    assert np.linalg.svd(q1.conj().T @ q2, compute_uv=False).min() > 1 - 1e-10


def test_cpqr_eigen_conventions():
    """Pivot order and the R diagonal follow Eigen's ColPivHouseholderQR:
    first column of largest norm, |R_kk| non-increasing for exact norms."""
    z = np.array([[1.0, 3.0, 3.0], [0.0, 0.0, 4.0]], complex)
    q, k, piv, rd = O.pivoted_qr_truncate(z, 1e-12)
    assert piv[0] == 2  # ||col2|| = 5 is the largest
    assert np.isclose(rd[0], 5.0)
    # beta = -sign(Re c0) ||x||: first Q column = -col/5 (c0 = 3 > 0)
    assert np.allclose(q[:, 0], -z[:, 2] / 5.0)
    # ties resolve to the first index
    q, k, piv, rd = O.pivoted_qr_truncate(np.eye(3, dtype=complex), 1e-12)
    assert list(piv) == [0, 1, 2]


def test_pinv_oracles():
    """test_linalg.cpp:180-200"""
    assert np.linalg.norm(O.pinv_solve(np.eye(3)) - np.eye(3)) < 1e-14
    d = np.zeros((2, 2))
    d[0, 0] = 2.0
    dp = O.pinv_solve(d)
    assert abs(dp[0, 0] - 0.5) < 1e-14 and abs(dp[1, 1]) < 1e-14
    m = O.gaussian_matrix(6, 4, 77, True)
    mp = O.pinv_solve(m)
    assert np.linalg.norm(mp @ m - np.eye(4)) < 1e-10
    ref = np.linalg.inv(m.T @ m) @ m.T
    assert np.linalg.norm(mp - ref) < 1e-10 * np.linalg.norm(ref)
    mc = O.gaussian_matrix(5, 3, 78)
    assert np.linalg.norm(mc @ O.pinv_solve(mc) @ mc - mc) < 1e-10 * np.linalg.norm(mc)
    assert rel_err(O.pinv_solve(mc), np.linalg.pinv(mc)) < 1e-12


def test_complex_orthonormality():
    """test_linalg.cpp:202-207"""
    q, k, _, _ = O.pivoted_qr_truncate(O.gaussian_matrix(12, 6, 90), 1e-12)
    assert k == 6
    assert np.linalg.norm(q.conj().T @ q - np.eye(6)) <= 1e-12 * np.sqrt(6)


# ------------------------------------------------------------- butterfly
def test_synth_invariants_and_dense_apply():
    """test_butterfly.cpp:45-108"""
    for real in (True, False):
        bf = O.synth_butterfly(3, 2, 5, real=real)
        assert bf.rows == 64
        d = bf.to_dense()
        x = O.gaussian_matrix(64, 3, 1, real)
        assert rel_err(bf.apply(x), d @ x) < 1e-12
        assert rel_err(bf.apply_adjoint(x), d.conj().T @ x) < 1e-12
        assert rel_err(bf.apply_transpose(x), d.T @ x) < 1e-12


def test_nnz_closed_form():
    """test_butterfly.cpp:118-132: nnz = 2^L (8r + 8r + r^2) + (L) 2^L 2r^2"""
    for L, r in ((4, 2), (5, 4)):
        bf = O.synth_butterfly(L, r, 1)
        nb = 1 << L
        assert bf.nnz() == nb * (8 * r + 8 * r + r * r) + L * nb * 2 * r * r


def test_container_round_trip_and_errors():
    """test_butterfly.cpp:159-210"""
    bf = O.synth_butterfly(4, 3, 2)
    data = bf.serialize()
    assert data[:4] == b"BFH1"
    back = O.HybridButterfly.deserialize(data)
    assert back.serialize() == data
    with pytest.raises(O.OracleError):
        O.HybridButterfly.deserialize(data[: len(data) // 2])
    bad = bytearray(data)
    bad[0] ^= 0xFF
    with pytest.raises(O.OracleError):
        O.HybridButterfly.deserialize(bytes(bad))


# ------------------------------------------------------------ reconstruct
def test_structured_probes_slice_columns():
    """test_reconstruct.cpp:32-67"""
    a = O.gaussian_matrix(32, 32, 3, True)
    op = O.dense_operator(a, real=True)
    t = O.PartitionTree.build(np.arange(32, dtype=float), 3)
    core = O.gaussian_matrix(4, 4, 9, True)
    res = O.probe_with(op, t, 3, 5, core, forward=True)
    b, e = t.node_range(3, 5)
    assert rel_err(res, a[:, b:e] @ core) <= 1e-13
    assert op.counters()[0] == 4
    O.probe_with(op, t, 3, 1, O.gaussian_matrix(4, 2, 9, True), forward=False)
    assert op.counters()[1] == 2
    with pytest.raises(O.OracleError):
        O.probe_with(op, t, 3, 0, np.zeros((3, 2)))


def test_core_block_fit():
    """test_reconstruct.cpp:69-107"""
    u = O.householder_q(O.gaussian_matrix(16, 4, 1, True))
    v = O.householder_q(O.gaussian_matrix(16, 4, 2, True))
    bt = O.gaussian_matrix(4, 4, 3, True)
    k = u @ bt @ v.T
    om = O.gaussian_matrix(16, 6, 4, True)
    b = O.core_block(k @ om, u, v.T @ om)
    assert np.linalg.norm(b - bt) <= 1e-10 * np.linalg.norm(bt)
    # local optimality
    u = O.householder_q(O.gaussian_matrix(12, 3, 8, True))
    v = O.householder_q(O.gaussian_matrix(12, 3, 9, True))
    k = O.gaussian_matrix(12, 12, 10, True)
    om = O.gaussian_matrix(12, 5, 11, True)
    coeff = v.T @ om
    b = O.core_block(k @ om, u, coeff)
    best = np.linalg.norm(k @ om - u @ b @ coeff)
    for trial in range(20):
        pb = b + 1e-3 * O.gaussian_matrix(3, 3, 100 + trial, True)
        assert best <= np.linalg.norm(k @ om - u @ pb @ coeff) + 1e-10
    with pytest.raises(O.OracleError):
        O.core_block(O.gaussian_matrix(8, 3, 14, True), O.householder_q(O.gaussian_matrix(8, 4, 12, True)),
                     O.gaussian_matrix(4, 3, 13, True))


@pytest.mark.parametrize("real,L,r,seed", [(True, 5, 8, 7), (False, 4, 4, 21)])
def test_synthetic_exact_recovery(real, L, r, seed):
    """test_reconstruct.cpp:109-157"""
    bf0 = O.synth_butterfly(L, r, seed, real=real)
    n = (1 << L) * 8
    op = O.butterfly_operator(bf0)
    t = O.PartitionTree.build(np.arange(n, dtype=float), L)
    bf, log = O.factorize(op, t, t, dict(levels=L, tolerance=1e-10, rank_guess=4, oversampling=2, seed=seed + 1000))
    f, tr = op.counters()
    assert sum(p["forward_columns"] + p["transpose_columns"] for p in log["phases"]) == f + tr
    assert O.estimate_error(op, bf, 16, 1 if real else 2) <= 1e-10
    assert (bf.rank_profile() == r).all()
    if r == 8:
        ph = {p["name"]: p for p in log["phases"]}
        assert ph["leaf_v"]["rounds"] == 2
        assert ph["leaf_v"]["transpose_columns"] == 6 + 10 + 18
        assert ph["leaf_u"]["forward_columns"] == 6 + 10 + 18
        for l in range(L - 1, L // 2 - 1, -1):
            assert ph[f"transfer_r_{l}"]["forward_columns"] == (1 << (L - l)) * (2 * 8 + 2)
        for l in range(1, L // 2 + 1):
            assert ph[f"transfer_w_{l}"]["transpose_columns"] == (1 << l) * (2 * 8 + 2)
    assert log["peak_concurrent_probes"] == 1 and log["peak_probe_bytes"] > 0


def test_zero_operator():
    """test_reconstruct.cpp:159-169"""
    op = O.dense_operator(np.zeros((64, 64)), real=True)
    t = O.PartitionTree.build(np.arange(64, dtype=float), 3)
    bf, log = O.factorize(op, t, t, dict(levels=3, tolerance=1e-8))
    assert bf.max_rank() == 0
    assert log["phases"][0]["rounds"] == 0
    with pytest.raises(O.OracleError) as e:
        O.estimate_error(op, bf)
    assert e.value.code == 5


def test_phase_sequencing():
    """test_reconstruct.cpp:171-196"""
    bf0 = O.synth_butterfly(4, 2, 3, real=True)
    op = O.butterfly_operator(bf0)
    t = O.PartitionTree.build(np.arange(128, dtype=float), 4)
    cfg = dict(levels=4, tolerance=1e-10, rank_guess=4, oversampling=2, seed=1003)
    f = O.Factorizer(op, t, t, cfg)
    with pytest.raises(O.OracleError):
        f.transfer_level_w(1)
    f.leaf_row_bases()
    with pytest.raises(O.OracleError):
        f.leaf_row_bases()
    f.leaf_col_bases()
    with pytest.raises(O.OracleError):
        f.transfer_level_r(3)
    with pytest.raises(O.OracleError):
        f.transfer_level_w(2)
    f.transfer_level_w(1)
    f.transfer_level_w(2)
    with pytest.raises(O.OracleError):
        f.transfer_level_r(2)
    f.transfer_level_r(3)
    f.transfer_level_r(2)
    assert f.complete()


def test_byte_identical_across_runs_and_threads():
    """test_reconstruct.cpp:198-209"""
    bf0 = O.synth_butterfly(4, 4, 11, real=True)
    op = O.butterfly_operator(bf0)
    t = O.PartitionTree.build(np.arange(128, dtype=float), 4)
    cfg = dict(levels=4, tolerance=1e-10, rank_guess=4, oversampling=2, seed=1011)
    a, _ = O.factorize(op, t, t, cfg)
    b, _ = O.factorize(op, t, t, cfg)
    c, _ = O.factorize(op, t, t, dict(cfg, threads=4))
    assert a.serialize() == b.serialize() == c.serialize()


def test_literal_transpose_core_worse():
    """test_reconstruct.cpp:211-221"""
    bf0 = O.synth_butterfly(4, 4, 31, real=True)
    op = O.butterfly_operator(bf0)
    t = O.PartitionTree.build(np.arange(128, dtype=float), 4)
    cfg = dict(levels=4, tolerance=1e-10, rank_guess=4, oversampling=2, seed=1031)
    good, _ = O.factorize(op, t, t, cfg)
    lit, _ = O.factorize(op, t, t, dict(cfg, literal_transpose_core=1))
    eg, el = O.estimate_error(op, good, 16, 5), O.estimate_error(op, lit, 16, 5)
    assert eg <= 1e-10 and el > eg


def test_tolerance_monotone_on_plates(oracle_threads):
    """test_reconstruct.cpp:246-269 analogue on the config-1 kernel."""
    op, rt, ct, cfg = oracle_config(1, 256)

    def med(eps):
        errs = []
        for s in range(3):
            bf, _ = O.factorize(op, rt, ct, dict(cfg, tolerance=eps, seed=s, rank_guess=4, threads=oracle_threads))
            errs.append(O.estimate_error(op, bf, 16, s + 50))
        return sorted(errs)[1]

    assert med(1e-3) <= med(1e-2) + 1e-12


@pytest.mark.parametrize("cfg_id,n", [(0, 512), (1, 256), (2, 1024), (4, 1024)])
def test_configs_reach_tolerance(oracle_threads, cfg_id, n):
    """Every BASELINE operator is factorized to ~tol by the oracle."""
    op, rt, ct, cfg = oracle_config(cfg_id, n)
    bf, log = O.factorize(op, rt, ct, dict(cfg, threads=oracle_threads))
    err = O.estimate_error(op, bf, 16, 0)
    assert err < 50 * cfg["tolerance"], err
    if cfg_id == 4:
        assert bf.max_rank() == 32
