"""Butterfly apply at k <= 2 columns (the PDL-chained stage kernels,
k_gemm.cu bgemm_stage_kernel -- HybridButterfly::apply / apply_adjoint /
apply_transpose, butterfly.hpp:71-193) against the CPU oracle, on synthetic
butterflies and a factorization with ragged ranks and leaves, across repeated
and interleaved calls (CUDA-graph replays)."""
import numpy as np
import pytest

import oracle as O
from helpers import rel_err

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def A():
    import paper_2002_03400_b200.api as A

    return A


def _pair(A, levels, rank, seed, leaf):
    bf = A.synth_butterfly(levels, rank, seed, leaf=leaf, perturb=1e-8)
    return bf, O.HybridButterfly.deserialize(bytes(bf.serialize()))


@pytest.mark.parametrize("levels,rank,leaf", [(4, 4, 8), (7, 8, 16), (10, 16, 32)])
@pytest.mark.parametrize("k", [1, 2])
def test_small_k_apply_matches_oracle(A, levels, rank, leaf, k):
    bf, bo = _pair(A, levels, rank, 3, leaf)
    rng = np.random.default_rng(levels * 10 + k)
    x = np.asfortranarray(rng.standard_normal((bf.cols, k)) + 1j * rng.standard_normal((bf.cols, k)))
    y = np.asfortranarray(rng.standard_normal((bf.rows, k)) + 1j * rng.standard_normal((bf.rows, k)))
    ref_n, ref_h, ref_t = bo.apply(x), bo.apply_adjoint(y), bo.apply_transpose(y)
    first_n, first_h = bf.apply(x), bf.apply_adjoint(y)
    assert rel_err(first_n, ref_n) <= 1e-12
    assert rel_err(first_h, ref_h) <= 1e-12
    assert rel_err(bf.apply_transpose(y), ref_t) <= 1e-12
    # repeated and interleaved calls (graph replays, flag generations)
    for _ in range(4):
        np.testing.assert_array_equal(bf.apply(x), first_n)
        np.testing.assert_array_equal(bf.apply_adjoint(y), first_h)


def test_small_k_apply_factorized(A):
    """A factorization with adaptive (ragged) ranks and ragged leaves."""
    import paper_2002_03400_b200 as B

    w = B.configs.build(0, 1000)
    bf, _ = B.factorize(w.op, w.row_tree, w.col_tree, w.recon)
    bo = O.HybridButterfly.deserialize(bytes(bf.serialize()))
    rng = np.random.default_rng(0)
    for k in (1, 2):
        x = np.asfortranarray(rng.standard_normal((bf.cols, k)) + 1j * rng.standard_normal((bf.cols, k)))
        assert rel_err(bf.apply(x), bo.apply(x)) <= 1e-12
        assert rel_err(bf.apply_adjoint(x[: bf.rows]), bo.apply_adjoint(x[: bf.rows])) <= 1e-12
