"""Process layouts of the apply (reference inc/layout.hpp; tests/test_layout.cpp
and acceptance criterion 6 are the model).

CPU: the oracle restatement (oracle/layout_oracle.py) and the library's
host-only entry points (bfly_comm_cost, bfly_layout_owners) reproduce the
reference's comm_cost grid, rejected specs, ownership maps and simulated
sweep tallies stored in tests/golden/layout.npz (made from oracle/_ref).
GPU: the distributed apply (bfly_apply_layout, p virtual processes on one
GPU through the same transfer plan, pack and unpack kernels a multi-GPU run
uses) is bit-identical to the single-GPU apply and reports the reference's
tallies; on the synthetic butterflies they equal the closed-form model.
"""
import os

import numpy as np
import pytest

import layout_oracle as LO

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
KINDS = ("column", "row", "hybrid")


def _g():
    return np.load(os.path.join(GOLDEN, "layout.npz"))


@pytest.fixture(scope="module")
def A():
    import paper_2002_03400_b200.api as A

    return A


# ------------------------------------------------------------------ oracle --
def test_oracle_comm_cost_golden():
    g = _g()
    for (kind, L, r, p), v in zip(g["cc_spec"], g["cc_val"]):
        assert LO.comm_cost(int(kind), int(L), int(r), int(p)) == list(v), (kind, L, r, p)
    for kind, L, r, p in g["cc_bad"]:
        with pytest.raises(ValueError):
            LO.comm_cost(int(kind), int(L), int(r), int(p))


def test_oracle_owners_golden():
    g = _g()
    for tag, L in (("synth4", 4), ("synth6", 6), ("cfg0", int(g["cfg0_L"]))):
        for (kind, p), own in zip(g[f"{tag}_spec"], g[f"{tag}_owners"]):
            np.testing.assert_array_equal(LO.owners(int(kind), L, L // 2, int(p)).ravel(), own, err_msg=f"{tag} {kind} {p}")


def test_oracle_synth_tallies_match_reference_and_model():
    """Acceptance criterion 6: the simulated sweep equals the closed form on
    the constant-rank synthetic butterflies."""
    g = _g()
    const8 = lambda l, tau, nu: 8  # noqa: E731  (synth_butterfly: rank 8 everywhere)
    for L in (4, 6):
        n = 8 << L
        for (kind, p), t in zip(g[f"synth{L}_spec"], g[f"synth{L}_tally"]):
            got = LO.simulated_tallies(int(kind), L, L // 2, int(p), const8, const8, n, n)
            assert got == list(t), (L, kind, p)
            assert got == LO.comm_cost(int(kind), L, 8, int(p)), (L, kind, p)


# ------------------------------------------------- library (host entries) --
def test_native_comm_cost_golden(A):
    g = _g()
    for (kind, L, r, p), v in zip(g["cc_spec"], g["cc_val"]):
        rep = A.comm_cost(A.LayoutSpec(KINDS[kind], int(L), int(r), int(p)))
        assert [rep.exchange_volume, rep.exchange_msgs, rep.alltoall_volume, rep.alltoall_msgs] == list(v)
    for kind, L, r, p in g["cc_bad"]:
        with pytest.raises(A.PreconditionError):
            A.comm_cost(A.LayoutSpec(KINDS[kind], int(L), int(r), int(p)))
    with pytest.raises(A.PreconditionError):
        A.layout_from_name("diagonal")


def test_native_ownership_golden(A):
    g = _g()
    for tag, L in (("synth4", 4), ("synth6", 6), ("cfg0", int(g["cfg0_L"]))):
        for (kind, p), own in zip(g[f"{tag}_spec"], g[f"{tag}_owners"]):
            m = A.assign_ownership((L, L // 2), A.LayoutSpec(KINDS[kind], L, 1, int(p)))
            flat = np.concatenate([m.u_leaf, m.v_leaf, m.r_owner.ravel(), m.w_owner.ravel(), m.b_owner])
            np.testing.assert_array_equal(flat, own, err_msg=f"{tag} {kind} {p}")
    with pytest.raises(A.DimensionError):
        A.assign_ownership((4, 2), A.LayoutSpec("hybrid", 5, 4, 2))


def test_native_model_properties(A):
    """tests/test_layout.cpp sections: hybrid exchange-free while p^2 <= 2^L,
    oversubscribed hybrid pays 2g - L, row == column by symmetry, hybrid never
    exceeds column, model_time monotone."""
    for L in (4, 6, 8):
        for g in range(L + 1):
            p = 1 << g
            h = A.comm_cost(A.LayoutSpec("hybrid", L, 8, p))
            c = A.comm_cost(A.LayoutSpec("column", L, 8, p))
            r = A.comm_cost(A.LayoutSpec("row", L, 8, p))
            assert h.exchange_volume <= c.exchange_volume
            assert (c.exchange_volume, c.alltoall_volume) == (r.exchange_volume, r.alltoall_volume)
            if p * p <= (1 << L):
                assert h.exchange_msgs == 0 and h.exchange_volume == 0.0
            else:
                assert h.exchange_msgs == 2 * g - L
    rep = A.comm_cost(A.LayoutSpec("column", 6, 4, 8))
    assert rep.model_time(2.0, 1.0) > rep.model_time(1.0, 1.0) and rep.model_time(1.0, 2.0) > rep.model_time(1.0, 1.0)


# --------------------------------------------------------------------- GPU --
def _layout_vs_plain(A, bf, L, spec_list, golden_tallies, k=3, seed=11):
    rng = np.random.default_rng(seed)
    x = rng.standard_normal((bf.cols, k)) + 1j * rng.standard_normal((bf.cols, k))
    yh = rng.standard_normal((bf.rows, k)) + 1j * rng.standard_normal((bf.rows, k))
    y0 = bf.apply(x)
    x0 = bf.apply_adjoint(yh)
    moved = {}
    for (kind, p), t in zip(spec_list, golden_tallies):
        spec = A.LayoutSpec(KINDS[kind], L, 1, int(p))
        y, rep, mv = bf.apply_layout(x, spec)
        np.testing.assert_array_equal(y, y0, err_msg=f"{KINDS[kind]} p={p}")
        xa, rep_h, _ = bf.apply_layout(yh, spec, trans=A.H)
        np.testing.assert_array_equal(xa, x0, err_msg=f"adjoint {KINDS[kind]} p={p}")
        got = [rep.exchange_volume, rep.exchange_msgs, rep.alltoall_volume, rep.alltoall_msgs]
        assert got == list(t), (KINDS[kind], p, got, list(t))
        if p == 1:
            assert mv["total_recv"] == 0.0
        moved[(kind, int(p))] = mv["total_recv"]
    return moved


@pytest.mark.gpu
@pytest.mark.parametrize("L", [4, 6])
def test_gpu_layout_apply_synth(A, L):
    g = _g()
    bf = A.synth_butterfly(L, 8, L)
    spec = g[f"synth{L}_spec"]
    moved = _layout_vs_plain(A, bf, L, spec, g[f"synth{L}_tally"])
    for (kind, p), t in zip(spec, g[f"synth{L}_tally"]):
        m = A.comm_cost(A.LayoutSpec(KINDS[kind], L, 8, int(p)))
        assert [m.exchange_volume, m.exchange_msgs, m.alltoall_volume, m.alltoall_msgs] == list(t)
    for g_ in range(1, L + 1):
        p = 1 << g_
        if p * p <= (1 << L):
            # exchange-free hybrid: only the centre handoff moves data, each
            # centre coefficient block at most once (u_state(center) = 8 2^L)
            assert 0 < moved[(2, p)] <= 8 << L


@pytest.mark.gpu
def test_gpu_layout_apply_factorized(A):
    """The config-0 n=1024 factorization (ranks from the adaptive loop):
    tallies equal the reference's simulated sweep on its own factorization."""
    import paper_2002_03400_b200 as B

    g = _g()
    d = np.load(os.path.join(GOLDEN, "cfg0_n1024.npz"))
    L = int(d["L"])
    rt = B.PartitionTree.build(d["rows_pts"][:, :1], L, 1)
    ct = B.PartitionTree.build(d["cols_pts"][:, :1], L, 1)
    op = B.NufftOperator(d["rows_pts"], d["cols_pts"])
    rc = B.ReconstructionConfig(tolerance=float(d["tol"]), rank_guess=int(d["r0"]), levels=L, seed=int(d["seed"]))
    bf, _ = B.factorize(op, rt, ct, rc)
    np.testing.assert_array_equal(bf.rank_profile(), d["rank_profile"])
    _layout_vs_plain(A, bf, L, g["cfg0_spec"], g["cfg0_tally"], k=2)


@pytest.mark.gpu
def test_gpu_layout_rejects(A):
    bf = A.synth_butterfly(4, 4, 1)
    x = np.ones((bf.cols, 1), complex)
    with pytest.raises(A.PreconditionError):
        bf.apply_layout(x, A.LayoutSpec("hybrid", 4, 1, 3))
    with pytest.raises(A.PreconditionError):
        bf.apply_layout(x, A.LayoutSpec("hybrid", 4, 1, 32))
    with pytest.raises(A.DimensionError):
        bf.apply_layout(x, A.LayoutSpec("hybrid", 5, 1, 2))
    with pytest.raises(A.PreconditionError):
        bf.apply_layout(x, A.LayoutSpec("hybrid", 4, 1, 2), trans=A.T)
