"""BASELINE configs at their FULL sizes on the GPU, through size-independent
properties -- a complement to tests/test_full_parity.py, which compares the
full-size factorizations with fixtures frozen from the reference / oracle runs
(minutes of CPU time per config on the GPU box's host, too slow to repeat in
the test suite):

* the black box itself: sampled output rows / columns of the GPU products
  (int8-slice tensor-core K2 at full size) against the oracle's kernel
  operator restricted to those rows (operators.hpp:430-439 pattern);
* the factorization: the randomized error estimate (reconstruct.hpp:423-434)
  at the tolerance level, adjoint consistency <y, B x> = <B^H y, x>,
  linearity, and a .bfh round trip that reproduces apply bit for bit;
* config 4 (recompression of a rank-32 butterfly): every block rank exactly
  32 and the recompressed operator equal to the input one to 1e-12;
* the sharded schedule (8 virtual ranks, split probes at levels 1-2) equal to
  the single-GPU factorization at full size.
"""
import numpy as np
import pytest

import oracle as O
from helpers import oracle_points, rel_err

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def B():
    import paper_2002_03400_b200 as B

    return B


_CACHE = {}


def _factorized(B, cfg_id):
    if cfg_id not in _CACHE:
        w = B.configs.build(cfg_id)
        bf, log = B.factorize(w.op, w.row_tree, w.col_tree, w.recon)
        _CACHE[cfg_id] = (w, bf, log)
    return _CACHE[cfg_id]


@pytest.mark.parametrize("cfg_id", [1, 2])
def test_full_size_black_box_rows_match_oracle(B, cfg_id):
    w = B.configs.build(cfg_id)
    n = w.op.rows
    t, s, kind, kappa = oracle_points(cfg_id, n)
    rng = np.random.default_rng(cfg_id)
    rows = np.sort(rng.choice(n, 24, replace=False))
    cols = np.sort(rng.choice(n, 24, replace=False))
    x = O.gaussian_matrix(n, 4, O.seed_mix(7, 1))
    y = O.gaussian_matrix(n, 4, O.seed_mix(7, 2))
    # forward: rows of K x
    got = w.op.apply(x)[rows]
    ref = O.kernel_operator(kind, np.ascontiguousarray(t[rows]), s, kappa).apply(x)
    assert rel_err(got, ref) <= 1e-12
    # adjoint: rows of K^H y are columns of K
    got_h = w.op.apply_adjoint(y)[cols]
    ref_h = O.kernel_operator(kind, t, np.ascontiguousarray(s[cols]), kappa).apply_adjoint(y)
    assert rel_err(got_h, ref_h) <= 1e-12


@pytest.mark.parametrize("cfg_id", [1, 2])
def test_full_size_factorization_properties(B, cfg_id):
    w, bf, log = _factorized(B, cfg_id)
    tol = w.recon.tolerance
    # sampled relative error of the factorization through the GPU black box
    err = B.estimate_error(w.op, bf, 16, 3)
    assert 0.0 < err <= 10 * tol, err
    prof = bf.rank_profile()
    assert prof.min() >= 1 and prof.max() == bf.max_rank()
    # apply: adjoint consistency and linearity
    x = O.gaussian_matrix(bf.cols, 3, O.seed_mix(9, 1))
    y = O.gaussian_matrix(bf.rows, 3, O.seed_mix(9, 2))
    bx, bhy = bf.apply(x), bf.apply_adjoint(y)
    lhs, rhs = np.vdot(y, bx), np.vdot(bhy, x)
    assert abs(lhs - rhs) <= 1e-12 * abs(lhs)
    x2 = O.gaussian_matrix(bf.cols, 3, O.seed_mix(9, 3))
    assert rel_err(bf.apply(x + 2.0 * x2), bx + 2.0 * bf.apply(x2)) <= 1e-13
    # .bfh round trip: the same operator bit for bit
    bf2 = B.HybridButterfly.deserialize(bytes(bf.serialize()))
    np.testing.assert_array_equal(bf2.rank_profile(), prof)
    np.testing.assert_array_equal(bf2.apply(x), bx)
    # bookkeeping: every transfer phase multiplied probes of width max(r1+r2)+p
    for p in log.phases:
        if p.name.startswith("transfer"):
            assert p.probe_width >= 3 and (p.forward_columns > 0) != (p.transpose_columns > 0)


def test_full_size_recompression_exact_ranks(B):
    w, bf, log = _factorized(B, 4)
    assert (bf.rank_profile() == 32).all()
    x = O.gaussian_matrix(bf.cols, 4, O.seed_mix(11, 1))
    assert rel_err(bf.apply(x), w.op.apply(x)) <= 1e-12
    y = O.gaussian_matrix(bf.rows, 4, O.seed_mix(11, 2))
    assert rel_err(bf.apply_adjoint(y), w.op.apply_adjoint(y)) <= 1e-12
    assert B.estimate_error(w.op, bf, 16, 1) <= 1e-12


@pytest.mark.parametrize("cfg_id", [2, 4])
def test_full_size_sharded_schedule_matches(B, cfg_id):
    import dataclasses

    w, a, la = _factorized(B, cfg_id)
    b, lb = B.factorize(w.op, w.row_tree, w.col_tree, dataclasses.replace(w.recon, virtual_ranks=8))
    np.testing.assert_array_equal(a.rank_profile(), b.rank_profile())
    x = O.gaussian_matrix(w.op.cols, 4, 31)
    assert rel_err(b.apply(x), a.apply(x)) < 1e-12
    for pa, pb in zip(la.phases, lb.phases):
        if pa.name.startswith("transfer"):
            assert (pa.forward_columns, pa.transpose_columns) == (pb.forward_columns, pb.transpose_columns)
        assert pa.rounds == pb.rounds and pa.probe_width == pb.probe_width
