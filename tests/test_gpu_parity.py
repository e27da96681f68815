"""GPU parity: the sm_100a construction path against the CPU oracle.

Bar (BASELINE north_star): identical per-level rank profiles, identical
phase bookkeeping (columns, rounds, widths), and butterfly-apply outputs on
seeded probes within 1e-10 relative (complex128).  Cases follow the
reference's own tests (tests/test_reconstruct.cpp) plus every BASELINE
config at sizes the oracle finishes in seconds.
"""
import numpy as np
import pytest

import oracle as O
from helpers import oracle_config, rel_err

pytestmark = pytest.mark.gpu

APPLY_TOL = 1e-10


@pytest.fixture(scope="module")
def B():
    import paper_2002_03400_b200 as B

    return B


def _compare(bf_gpu, log_gpu, bf_or, log_or, n_rows, n_cols, seed=5, real=False, tol=APPLY_TOL):
    # rank profiles: every block of every level
    np.testing.assert_array_equal(bf_gpu.rank_profile(), bf_or.rank_profile())
    # phase bookkeeping (reconstruct.hpp:87-120)
    names = [p.name for p in log_gpu.phases]
    assert names == [p["name"] for p in log_or["phases"]]
    for pg, po in zip(log_gpu.phases, log_or["phases"]):
        assert pg.forward_columns == po["forward_columns"], pg.name
        assert pg.transpose_columns == po["transpose_columns"], pg.name
        assert pg.rounds == po["rounds"], pg.name
        assert pg.probe_width == po["probe_width"], pg.name
    assert log_gpu.rank_capped == log_or["rank_capped"]
    # apply outputs on seeded probes
    x = O.gaussian_matrix(n_cols, 16, O.seed_mix(seed, 5), real=real)
    y = O.gaussian_matrix(n_rows, 16, O.seed_mix(seed, 6), real=real)
    e_n = rel_err(bf_gpu.apply(x), bf_or.apply(x))
    e_h = rel_err(bf_gpu.apply_adjoint(y), bf_or.apply_adjoint(y))
    e_t = rel_err(bf_gpu.apply_transpose(y), bf_or.apply_transpose(y))
    assert e_n <= tol and e_h <= tol and e_t <= tol, (e_n, e_h, e_t)
    return e_n, e_h


def _run_config(B, cfg_id, n, oracle_threads):
    op_o, rt_o, ct_o, cfg = oracle_config(cfg_id, n)
    bf_o, log_o = O.factorize(op_o, rt_o, ct_o, dict(cfg, threads=oracle_threads))
    w = B.configs.build(cfg_id, n)
    assert np.array_equal(w.row_tree.perm, rt_o.perm) and np.array_equal(w.col_tree.flat_ranges, ct_o.range_flat)
    bf_g, log_g = B.factorize(w.op, w.row_tree, w.col_tree, w.recon)
    errs = _compare(bf_g, log_g, bf_o, log_o, w.op.rows, w.op.cols)
    # sampled error of the GPU factorization through the GPU black box
    e_gpu = B.estimate_error(w.op, bf_g, 16, 3)
    e_or = O.estimate_error(op_o, bf_o, 16, 3)
    assert abs(e_gpu - e_or) <= 1e-3 * e_or + 1e-12
    return errs, e_gpu


def test_black_box_products_match_oracle(B, oracle_threads):
    """K2: every kernel operator, N / T / H, dense and structured probes."""
    for cfg_id, n in ((0, 1024), (1, 1024), (2, 1024), (3, 512)):
        op_o, rt, ct, _ = oracle_config(cfg_id, n)
        w = B.configs.build(cfg_id, n)
        x = O.gaussian_matrix(n, 7, 11)
        for name, fo, fg in (("N", op_o.apply, w.op.apply), ("T", op_o.apply_transpose, w.op.apply_transpose),
                             ("H", op_o.apply_adjoint, w.op.apply_adjoint)):
            e = rel_err(fg(x), fo(x))
            assert e < 1e-12, (cfg_id, name, e)
        # structured probe: only one node's rows nonzero
        xs = np.zeros_like(x)
        b, e_ = rt.node_range(2, 1)
        xs[b:e_] = x[b:e_]
        assert rel_err(w.op.apply_adjoint(xs), op_o.apply_adjoint(xs)) < 1e-12


@pytest.mark.parametrize("ncols", [33, 34, 40, 45, 48])
def test_pair_products_match_oracle(B, oracle_threads, ncols):
    """K2 on CTA pairs (probe tiles of 33..40 columns, and 41..48 for the 3D
    plates: one evaluation shared through DSMEM, diagonal blocks split between
    the two CTAs) vs the oracle, every kernel operator, N / T / H, dense and
    structured probes; and against the single-CTA tile path of the library."""
    import os
    cases = ((0, 1024), (1, 1024), (2, 2048), (3, 512)) if ncols <= 40 else ((1, 1024), (1, 2304))
    for cfg_id, n in cases:
        op_o, rt, ct, _ = oracle_config(cfg_id, n)
        w = B.configs.build(cfg_id, n)
        x = O.gaussian_matrix(n, ncols, 17)
        for name, fo, fg in (("N", op_o.apply, w.op.apply), ("T", op_o.apply_transpose, w.op.apply_transpose),
                             ("H", op_o.apply_adjoint, w.op.apply_adjoint)):
            yg = fg(x)
            e = rel_err(yg, fo(x))
            assert e < 1e-12, (cfg_id, name, ncols, e)
            os.environ["BFLY_OZ_PAIR"] = "0"
            try:
                e2 = rel_err(yg, fg(x))
            finally:
                del os.environ["BFLY_OZ_PAIR"]
            assert e2 < 1e-13, (cfg_id, name, ncols, e2)
        xs = np.zeros_like(x)
        b, e_ = rt.node_range(2, 1)
        xs[b:e_] = x[b:e_]
        assert rel_err(w.op.apply_adjoint(xs), op_o.apply_adjoint(xs)) < 1e-12


@pytest.mark.parametrize("cfg_id, n", [(0, 1000), (2, 1500), (1, 1369)])
def test_pair_products_ragged_and_complex64(B, oracle_threads, cfg_id, n):
    """CTA-pair K2 at sizes that are not multiples of the 128-row tile (the
    last row block is partial; split-K ranges are ragged), and the complex64
    operators on the same path (1e-5 vs the complex128 oracle)."""
    op_o, rt, ct, _ = oracle_config(cfg_id, n)
    x = O.gaussian_matrix(n, 34, 23)
    w = B.configs.build(cfg_id, n)
    for fo, fg in ((op_o.apply, w.op.apply), (op_o.apply_adjoint, w.op.apply_adjoint)):
        assert rel_err(fg(x), fo(x)) < 1e-12
    w64 = B.configs.build(cfg_id, n, scalar=B.COMPLEX64)
    y64 = w64.op.apply(x.astype(np.complex64)).astype(np.complex128)
    assert rel_err(y64, op_o.apply(x)) < 1e-5


def test_gaussian_stream_matches_oracle(B):
    for seed in (0, 1, 123456789):
        for rows, cols in ((1, 1), (7, 3), (1000, 5)):
            g = B.gaussian_matrix(rows, cols, seed)
            o = O.gaussian_matrix(rows, cols, seed)
            assert np.max(np.abs(g - o)) <= 4e-15 * max(1.0, np.max(np.abs(o)))
            gr = B.gaussian_matrix(rows, cols, seed, scalar=B.REAL64)
            orr = O.gaussian_matrix(rows, cols, seed, real=True)
            assert np.max(np.abs(gr - orr)) <= 4e-15 * max(1.0, np.max(np.abs(orr)))


def test_cpqr_matches_oracle(B):
    rng = np.random.default_rng(0)
    for rows, cols, rank in ((32, 18, 18), (64, 66, 20), (104, 106, 50), (30, 10, 3), (8, 20, 8)):
        a = rng.standard_normal((rows, rank)) + 1j * rng.standard_normal((rows, rank))
        b = rng.standard_normal((rank, cols)) + 1j * rng.standard_normal((rank, cols))
        s = np.logspace(0, -12, rank)
        z = (a * s) @ b
        qo, ko, _, _ = O.pivoted_qr_truncate(z, 0.25e-6)
        qg = B.pivoted_qr_truncate(z, 0.25e-6)
        assert qg.shape[1] == ko
        # same span, same phase convention (Eigen's beta = -sign(Re c0)||x||)
        assert rel_err(qg, qo) < 1e-9
    z0 = np.zeros((5, 3), complex)
    assert B.pivoted_qr_truncate(z0, 1e-8).shape[1] == 0


def test_pinv_matches_oracle(B):
    rng = np.random.default_rng(1)
    for rows, cols in ((4, 6), (15, 32), (32, 66), (6, 4), (5, 3)):
        m = rng.standard_normal((rows, cols)) + 1j * rng.standard_normal((rows, cols))
        assert rel_err(B.pinv_solve(m), O.pinv_solve(m)) < 1e-12
    d = np.zeros((2, 2), complex)
    d[0, 0] = 2.0
    p = B.pinv_solve(d)
    assert abs(p[0, 0] - 0.5) < 1e-14 and abs(p[1, 1]) < 1e-14


@pytest.mark.parametrize("real,levels,rank,seed", [(True, 5, 8, 7), (False, 4, 4, 21), (False, 6, 2, 3)])
def test_synthetic_exact_recovery(B, real, levels, rank, seed):
    """test_reconstruct.cpp:109-157 on the GPU, checked against the oracle."""
    scalar = B.REAL64 if real else B.COMPLEX128
    bf_in_g = B.synth_butterfly(levels, rank, seed, scalar=scalar)
    bf_in_o = O.synth_butterfly(levels, rank, seed, real=real)
    n = (1 << levels) * 8
    op_g = B.ButterflyOperator(bf_in_g)
    op_o = O.butterfly_operator(bf_in_o)
    rt_g = B.PartitionTree.build(np.arange(n, dtype=float), levels)
    rt_o = O.PartitionTree.build(np.arange(n, dtype=float), levels)
    cfg = dict(levels=levels, tolerance=1e-10, rank_guess=4, oversampling=2, seed=seed + 1000)
    bf_g, log_g = B.factorize(op_g, rt_g, rt_g, B.ReconstructionConfig(**cfg))
    bf_o, log_o = O.factorize(op_o, rt_o, rt_o, cfg)
    assert log_g.forward_columns() + log_g.transpose_columns() == op_g.total_columns()
    _compare(bf_g, log_g, bf_o, log_o, n, n, real=real)
    assert B.estimate_error(op_g, bf_g, 16, 1) <= 1e-10
    assert (bf_g.rank_profile() == rank).all()
    if rank == 8:
        assert log_g.phase("leaf_v").rounds == 2
        assert log_g.phase("leaf_v").transpose_columns == (4 + 2) + (8 + 2) + (16 + 2)


@pytest.mark.parametrize("cfg_id,n", [(0, 4096), (1, 1024), (2, 4096), (3, 1024), (4, 4096)])
def test_config_parity(B, oracle_threads, cfg_id, n):
    """Every BASELINE config (config 0 at its full size) against the oracle."""
    (e_n, e_h), e = _run_config(B, cfg_id, n, oracle_threads)
    print(f"config {cfg_id} n={n}: apply rel diff {e_n:.2e} / adjoint {e_h:.2e}; sampled error {e:.2e}")


def test_zero_operator(B):
    """test_reconstruct.cpp:159-169."""
    op = B.DenseOperator(np.zeros((64, 64)))
    t = B.PartitionTree.build(np.arange(64, dtype=float), 3)
    bf, log = B.factorize(op, t, t, B.ReconstructionConfig(levels=3, tolerance=1e-8))
    assert bf.max_rank() == 0
    assert log.phase("leaf_v").rounds == 0
    with pytest.raises(B.ConditioningError):
        B.estimate_error(op, bf)


def test_phase_sequencing(B):
    """test_reconstruct.cpp:171-196."""
    bf = B.synth_butterfly(4, 2, 3, scalar=B.REAL64)
    op = B.ButterflyOperator(bf)
    t = B.PartitionTree.build(np.arange(128, dtype=float), 4)
    cfg = B.ReconstructionConfig(levels=4, tolerance=1e-10, seed=1003)
    f = B.Factorizer(op, t, t, cfg)
    with pytest.raises(B.SequencingError):
        f.transfer_level_w(1)
    f.leaf_row_bases()
    with pytest.raises(B.SequencingError):
        f.leaf_row_bases()
    f.leaf_col_bases()
    with pytest.raises(B.SequencingError):
        f.transfer_level_r(3)
    with pytest.raises(B.SequencingError):
        f.transfer_level_w(2)
    f.transfer_level_w(1)
    f.transfer_level_w(2)
    with pytest.raises(B.SequencingError):
        f.transfer_level_r(2)
    f.transfer_level_r(3)
    f.transfer_level_r(2)
    assert f.complete()
    bf2, _ = f.take()
    assert B.estimate_error(op, bf2, 16, 1) < 1e-10


def test_determinism_and_container_roundtrip(B):
    """test_reconstruct.cpp:198-209: byte-identical containers across runs."""
    bf = B.synth_butterfly(4, 4, 11, scalar=B.REAL64)
    op = B.ButterflyOperator(bf)
    t = B.PartitionTree.build(np.arange(128, dtype=float), 4)
    cfg = B.ReconstructionConfig(levels=4, tolerance=1e-10, seed=1011)
    a, _ = B.factorize(op, t, t, cfg)
    b, _ = B.factorize(op, t, t, cfg)
    assert a.serialize() == b.serialize()
    # container parses in the oracle (the reference format) and round-trips
    o = O.HybridButterfly.deserialize(a.serialize())
    assert o.serialize() == a.serialize()
    c = B.HybridButterfly.deserialize(a.serialize(), scalar=B.REAL64)
    assert c.serialize() == a.serialize()


def test_literal_transpose_core_is_worse(B):
    """test_reconstruct.cpp:211-221."""
    bf = B.synth_butterfly(4, 4, 31, scalar=B.REAL64)
    op = B.ButterflyOperator(bf)
    t = B.PartitionTree.build(np.arange(128, dtype=float), 4)
    good, _ = B.factorize(op, t, t, B.ReconstructionConfig(levels=4, tolerance=1e-10, seed=1031))
    lit, _ = B.factorize(op, t, t, B.ReconstructionConfig(levels=4, tolerance=1e-10, seed=1031,
                                                          literal_transpose_core=True))
    e_good, e_lit = B.estimate_error(op, good, 16, 5), B.estimate_error(op, lit, 16, 5)
    assert e_good <= 1e-10 and e_lit > e_good


def test_batched_probes_match_unbatched(B):
    """Probe batching is a scheduling knob: results are bit-identical."""
    w = B.configs.build(2, 2048)
    a, la = B.factorize(w.op, w.row_tree, w.col_tree, w.recon)
    import dataclasses

    rc = dataclasses.replace(w.recon, max_batch_probes=3)
    b, lb = B.factorize(w.op, w.row_tree, w.col_tree, rc)
    np.testing.assert_array_equal(a.rank_profile(), b.rank_profile())
    x = O.gaussian_matrix(2048, 4, 9)
    assert rel_err(a.apply(x), b.apply(x)) < 1e-13
    assert lb.peak_concurrent_probes <= 3 < la.peak_concurrent_probes


def test_dense_callback_operator(B):
    """User black box through the C-ABI callback (stream-ordered)."""
    import torch

    rng = np.random.default_rng(3)
    n = 256
    a = rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n))
    at = torch.tensor(a, dtype=torch.complex128, device="cuda")

    def fn(trans, x, ldx, y, ldy, k, stream):
        return _torch_apply(at, trans, x, ldx, y, ldy, k, stream)

    op = B.CallbackOperator(n, n, fn)
    x = O.gaussian_matrix(n, 3, 4)
    assert rel_err(op.apply(x), a @ x) < 1e-13
    assert rel_err(op.apply_transpose(x), a.T @ x) < 1e-13
    assert rel_err(op.apply_adjoint(x), a.conj().T @ x) < 1e-13


def _torch_apply(at, trans, x, ldx, y, ldy, k, stream):
    import torch

    n = at.shape[0]

    class _CAI:
        def __init__(self, ptr, shape, strides):
            self.__cuda_array_interface__ = {"data": (ptr, False), "shape": shape, "typestr": "<c16",
                                             "strides": strides, "version": 3}

    # stream-ordered: run on the library's stream
    with torch.cuda.stream(torch.cuda.ExternalStream(stream)):
        X = torch.as_tensor(_CAI(x, (n, k), (16, 16 * ldx)), device="cuda")
        Y = torch.as_tensor(_CAI(y, (n, k), (16, 16 * ldy)), device="cuda")
        A = at if trans == 0 else at.t()
        Y.copy_(A @ X)
    return 0


@pytest.mark.parametrize("cfg_id,n,vr", [(0, 2048, 2), (0, 2048, 3), (2, 4096, 8), (4, 4096, 4), (1, 1024, 5),
                                        (3, 1024, 4), (2, 4096, 6)])
def test_virtual_ranks_match_single_gpu(B, cfg_id, n, vr):
    """The rank-sharded schedule (leaf rows, W blocks in place, R/B blocks
    packed -> gathered -> unpacked; levels with fewer probes than ranks split
    a probe's partner nodes, i.e. its output rows) executed for `vr` ranks in
    one process reproduces the single-GPU factorization."""
    import dataclasses

    w = B.configs.build(cfg_id, n)
    a, la = B.factorize(w.op, w.row_tree, w.col_tree, w.recon)
    b, lb = B.factorize(w.op, w.row_tree, w.col_tree, dataclasses.replace(w.recon, virtual_ranks=vr))
    np.testing.assert_array_equal(a.rank_profile(), b.rank_profile())
    x = O.gaussian_matrix(w.op.cols, 8, 21)
    y = O.gaussian_matrix(w.op.rows, 8, 22)
    assert rel_err(b.apply(x), a.apply(x)) < 1e-12
    assert rel_err(b.apply_adjoint(y), a.apply_adjoint(y)) < 1e-12
    assert [p.name for p in la.phases] == [p.name for p in lb.phases]
    for pa, pb in zip(la.phases, lb.phases):
        if pa.name.startswith("transfer"):
            assert (pa.forward_columns, pa.transpose_columns) == (pb.forward_columns, pb.transpose_columns)
        assert pa.rounds == pb.rounds and pa.probe_width == pb.probe_width


def test_complex64_recompression_vs_complex128_oracle(B, oracle_threads):
    """Config 4 at complex64 (B200-only variant; the reference has no complex64,
    core.hpp:29-39): checked against the complex128 oracle at 1e-4."""
    n = 4096
    w = B.configs.build(4, n, scalar=B.COMPLEX64)
    bf, log = B.factorize(w.op, w.row_tree, w.col_tree, w.recon)
    op_o, rt_o, ct_o, cfg = oracle_config(4, n)
    bf_o, _ = O.factorize(op_o, rt_o, ct_o, dict(cfg, threads=oracle_threads))
    x = O.gaussian_matrix(n, 16, O.seed_mix(5, 5))
    y_o = bf_o.apply(x)
    y_g = bf.apply(x.astype(np.complex64)).astype(np.complex128)
    assert rel_err(y_g, y_o) < 1e-4
    assert B.estimate_error(w.op, bf, 16, 1) < 1e-4
    assert bf.max_rank() <= 64


@pytest.mark.parametrize("cfg_id,n", [(0, 4096), (2, 4096), (4, 4096)])
def test_gpu_matches_reference_implementation(B, oracle_threads, cfg_id, n):
    """Directly against the reference implementation (oracle/_ref: the
    reference's own headers compiled against the Eigen-API shim)."""
    import refpy as R

    if not R.available():
        pytest.skip("oracle/_ref not built")
    from test_ref_pin import _ref_config

    R.lib().ref_set_threads(oracle_threads)
    op_r, L, tol, r0 = _ref_config(cfg_id, n)
    bf_r = R.factorize(op_r, tol, r0, L, seed=0, threads=oracle_threads)
    w = B.configs.build(cfg_id, n)
    bf_g, log_g = B.factorize(w.op, w.row_tree, w.col_tree, w.recon)
    np.testing.assert_array_equal(bf_g.rank_profile(), bf_r.rank_profile(L))
    phases_r, _ = bf_r.log()
    assert [(p.forward_columns, p.transpose_columns, p.rounds, p.probe_width) for p in log_g.phases] == phases_r
    x = O.gaussian_matrix(n, 16, O.seed_mix(9, 5))
    y = O.gaussian_matrix(n, 16, O.seed_mix(9, 6))
    assert rel_err(bf_g.apply(x), bf_r.apply(x, 0)) < APPLY_TOL
    assert rel_err(bf_g.apply_adjoint(y), bf_r.apply(y, 2)) < APPLY_TOL


def test_cpp_adapter_drop_in():
    """include/bfly_b200.hpp: the reference's own operators (synthetic real /
    complex, Helmholtz3D hemispheres) factorized on the GPU through the C-ABI
    callback from a C++ program built against the reference headers; ranks,
    bookkeeping and apply outputs equal the reference's CPU factorize()."""
    import os
    import subprocess

    exe = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "oracle", "_ref", "adapter_demo")
    if not os.path.exists(exe):
        pytest.skip("adapter demo not built (needs /root/reference at build time)")
    r = subprocess.run([exe], capture_output=True, text=True, timeout=600)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "ADAPTER PARITY OK" in r.stdout


def test_int8_range_fallback_recomputes_on_fp64(B, oracle_threads, monkeypatch):
    """K2's integer-slice path defers its range check to the end of a
    factorization; a flagged launch makes the whole factorization rerun on the
    FP64 DMMA path with the operator counters restored (forced here through
    the BFLY_OZ_TEST_OVERFLOW hook).  Results and bookkeeping must still be
    the oracle's, and the public apply path must recompute as well."""
    op_o, rt_o, ct_o, cfg = oracle_config(2, 1024)
    bf_o, log_o = O.factorize(op_o, rt_o, ct_o, dict(cfg, threads=oracle_threads))
    w = B.configs.build(2, 1024)
    monkeypatch.setenv("BFLY_OZ_TEST_OVERFLOW", "1")
    bf_g, log_g = B.factorize(w.op, w.row_tree, w.col_tree, w.recon)
    assert log_g.forward_columns() + log_g.transpose_columns() == w.op.total_columns()
    _compare(bf_g, log_g, bf_o, log_o, w.op.rows, w.op.cols)
    x = O.gaussian_matrix(w.op.cols, 3, 9)
    assert rel_err(w.op.apply(x), op_o.apply(x)) < 1e-12
    monkeypatch.delenv("BFLY_OZ_TEST_OVERFLOW")
    assert rel_err(w.op.apply(x), op_o.apply(x)) < 1e-12


@pytest.mark.parametrize("real", [False, True])
def test_serialize_into_caller_buffer_matches_oracle_layout(B, real):
    """The .bfh export is packed on the GPU straight into the file layout
    (serialize.hpp:103-127); writing into a caller-provided (reused, pinned)
    buffer gives the same bytes as the default allocation, and both parse in
    the oracle into the same container."""
    import torch

    scalar = B.REAL64 if real else B.COMPLEX128
    bf = B.synth_butterfly(5, 3, 17, scalar=scalar)
    op = B.ButterflyOperator(bf)
    t = B.PartitionTree.build(np.arange(256, dtype=float), 5)
    a, _ = B.factorize(op, t, t, B.ReconstructionConfig(levels=5, tolerance=1e-10, seed=5))
    ref = bytes(a.serialize())
    n = a.serialized_size()
    assert n == len(ref)
    host = torch.empty(n + 4096, dtype=torch.uint8, pin_memory=True)
    for _ in range(2):  # reuse
        view = a.serialize(out=host.numpy())
        assert len(view) == n and bytes(view) == ref
    o = O.HybridButterfly.deserialize(ref)
    assert bytes(o.serialize()) == ref
    x = O.gaussian_matrix(256, 3, 4, real=real)
    assert rel_err(a.apply(x), o.apply(x)) < 1e-13


def test_rank_cap_and_rectangular_operator(B, oracle_threads):
    """Edge cases of the adaptive loop against the oracle: a hard rank cap that
    stops the leaf doubling (reconstruct.hpp:389-393, rank_capped set) and a
    rectangular operator (m != n, row and column trees of different sizes)."""
    m, n = 768, 1024
    x = np.zeros((m, 3))
    xi = np.zeros((n, 3))
    O.lib().bo_points_uniform(m, 7, 1, 0.0, 1.0, O._ptr(x))
    O.lib().bo_points_uniform(n, 7, 2, -n / 2.0, n / 2.0, O._ptr(xi))
    L = 4
    for cap in (-1, 8):
        rt_o = O.PartitionTree.build(x[:, :1], L)
        ct_o = O.PartitionTree.build(xi[:, :1], L)
        op_o = O.kernel_operator(O.OP_NUFFT, x, xi)
        cfg = dict(levels=L, tolerance=1e-6, rank_guess=4, oversampling=2, seed=3, hard_cap=cap,
                   threads=oracle_threads)
        bf_o, log_o = O.factorize(op_o, rt_o, ct_o, cfg)
        op = B.NufftOperator(x, xi)
        rt = B.PartitionTree.build(x[:, :1], L, 1)
        ct = B.PartitionTree.build(xi[:, :1], L, 1)
        rc = B.ReconstructionConfig(tolerance=1e-6, rank_guess=4, levels=L, seed=3, hard_cap=cap)
        bf, log = B.factorize(op, rt, ct, rc)
        assert (bf.rows, bf.cols) == (m, n)
        _compare(bf, log, bf_o, log_o, m, n)
        assert log.rank_capped == (1 if cap > 0 else 0)
        if cap > 0:
            # the cap stops the leaf doubling: leaf bases from the round with r = cap
            assert log.phase("leaf_v").probe_width == cap + 2
        # the sharded schedule with non-identity trees (column-split leaf products)
        import dataclasses

        bv, _ = B.factorize(op, rt, ct, dataclasses.replace(rc, virtual_ranks=3))
        np.testing.assert_array_equal(bv.rank_profile(), bf.rank_profile())
        xv = O.gaussian_matrix(n, 4, 77)
        assert rel_err(bv.apply(xv), bf.apply(xv)) < 1e-12


def test_repeated_factorizations_identical(B):
    """Many factorizations on one context (the pinned upload ring wraps
    several times, pool re-reservations, CUDA-graph applies): every result
    bit-identical to the first."""
    w = B.configs.build(2, 8192)
    bf0, _ = B.factorize(w.op, w.row_tree, w.col_tree, w.recon)
    x = O.gaussian_matrix(w.op.cols, 2, 5)
    y0 = bf0.apply(x)
    prof0 = bf0.rank_profile()
    for _ in range(12):
        bf, _ = B.factorize(w.op, w.row_tree, w.col_tree, w.recon)
        np.testing.assert_array_equal(bf.rank_profile(), prof0)
        np.testing.assert_array_equal(bf.apply(x), y0)


@pytest.mark.parametrize("cfg_id,n", [(0, 2048), (2, 4096)])
def test_complex64_kernel_configs_vs_complex128_oracle(B, oracle_threads, cfg_id, n):
    """complex64 on the kernel-evaluated operators (B200-only variant):
    apply within 1e-4 of the complex128 oracle factorization."""
    op_o, rt_o, ct_o, cfg = oracle_config(cfg_id, n)
    bf_o, _ = O.factorize(op_o, rt_o, ct_o, dict(cfg, threads=oracle_threads))
    w = B.configs.build(cfg_id, n, scalar=B.COMPLEX64)
    bf, _ = B.factorize(w.op, w.row_tree, w.col_tree, w.recon)
    x = O.gaussian_matrix(w.op.cols, 8, O.seed_mix(5, 5))
    y = bf.apply(x.astype(np.complex64)).astype(np.complex128)
    assert rel_err(y, bf_o.apply(x)) < 1e-4


@pytest.mark.parametrize("cfg_id,n,seed", [(0, 1536, 2), (1, 2304, 2), (2, 3000, 1), (4, 2048, 1)])
def test_other_seeds_and_sizes(B, oracle_threads, cfg_id, n, seed):
    """Probe seeds != 0 and non-power-of-two sizes (ragged trees): identical
    rank profiles and apply within 1e-10 of the oracle."""
    op_o, rt_o, ct_o, cfg = oracle_config(cfg_id, n, seed=seed)
    bf_o, log_o = O.factorize(op_o, rt_o, ct_o, dict(cfg, threads=oracle_threads))
    w = B.configs.build(cfg_id, n, seed=seed)
    bf, log = B.factorize(w.op, w.row_tree, w.col_tree, w.recon)
    _compare(bf, log, bf_o, log_o, w.op.rows, w.op.cols, seed=seed)


def test_ranged_callback_skips_zero_rows(B, oracle_threads):
    """bfly_apply_range_fn: a user black box told each structured
    probe's nonzero input rows multiplies only those (A[:, b:e] X[b:e]); the
    factorization equals the oracle's (ranks, bookkeeping, apply 1e-10) and the
    same matrix as a padded reference-style callback, while the transfer-level
    products touch |node| rows instead of n (reconstruct.hpp:72-85)."""
    import torch

    n = 1024
    op_o, rt_o, ct_o, cfg = oracle_config(2, n)
    a = op_o.apply(np.eye(n, dtype=np.complex128))  # dense K (tree order = identity)
    at = torch.tensor(a, dtype=torch.complex128, device="cuda")
    calls = []

    class _CAI:
        def __init__(self, ptr, shape, strides):
            self.__cuda_array_interface__ = {"data": (ptr, False), "shape": shape, "typestr": "<c16",
                                             "strides": strides, "version": 3}

    def ranged(trans, x, ldx, y, ldy, k, b, e, stream):
        calls.append((trans, k, b, e))
        with torch.cuda.stream(torch.cuda.ExternalStream(stream)):
            X = torch.as_tensor(_CAI(x, (n, k), (16, 16 * ldx)), device="cuda")
            Y = torch.as_tensor(_CAI(y, (n, k), (16, 16 * ldy)), device="cuda")
            A = at[:, b:e] if trans == 0 else at[b:e, :].t()
            Y.copy_(A @ X[b:e])
        return 0

    op = B.CallbackOperator(n, n, ranged, ranged=True)
    x = O.gaussian_matrix(n, 3, 4)
    assert rel_err(op.apply(x), a @ x) < 1e-13 and calls[-1] == (0, 3, 0, n)
    assert rel_err(op.apply_adjoint(x), a.conj().T @ x) < 1e-13
    calls.clear()
    L = cfg["levels"]
    rt = B.PartitionTree.build(np.arange(n, dtype=np.float64)[:, None], L)  # identity trees
    rc = B.ReconstructionConfig(tolerance=cfg["tolerance"], rank_guess=cfg["rank_guess"], levels=L)
    bf, log = B.factorize(op, rt, rt, rc)
    bf_o, log_o = O.factorize(op_o, rt_o, ct_o, dict(cfg, threads=oracle_threads))
    _compare(bf, log, bf_o, log_o, n, n)
    dense = B.DenseOperator(a)
    bf_d, _ = B.factorize(dense, rt, rt, rc)
    np.testing.assert_array_equal(bf.rank_profile(), bf_d.rank_profile())
    # one call per structured probe, each with its node's rows only
    lm = L // 2
    sizes = sorted({e - b for _, _, b, e in calls})
    assert sizes[-1] == n  # the leaf rounds' dense Gaussian probes
    assert all(s in sizes for s in (n >> l for l in range(1, lm + 1)))  # W level l: |T_tau| = n / 2^l
    rows_used = sum((e - b) * k for _, k, b, e in calls)
    rows_padded = sum(n * k for _, k, b, e in calls)
    assert rows_used < 0.6 * rows_padded
    print(f"ranged callback: {len(calls)} calls, {rows_used / rows_padded:.2f} of the padded rows multiplied")


def test_memory_guard_shrinks_batches_then_refuses(B, monkeypatch):
    """Memory guard (SURVEY 7 hard part 5): before each level allocates, its
    factor level and per-probe working set are sized from the children's ranks
    (the width rule of reconstruct.hpp:204-207, 257-260).  With little memory
    left the probe batch shrinks (results bit-identical); with too little for
    one probe the factorization is refused up front with the bytes needed."""
    w = B.configs.build(2, 16384)
    a, la = B.factorize(w.op, w.row_tree, w.col_tree, w.recon)
    monkeypatch.setenv("BFLY_MEM_AVAIL_GB", "0.12")
    b, lb = B.factorize(w.op, w.row_tree, w.col_tree, w.recon)
    np.testing.assert_array_equal(a.rank_profile(), b.rank_profile())
    x = O.gaussian_matrix(w.op.cols, 4, 17)
    np.testing.assert_array_equal(a.apply(x), b.apply(x))
    assert lb.peak_concurrent_probes < la.peak_concurrent_probes
    print(f"guarded batch: {lb.peak_concurrent_probes} probes (unguarded {la.peak_concurrent_probes})")
    monkeypatch.setenv("BFLY_MEM_AVAIL_GB", "0.001")
    with pytest.raises(B.PreconditionError, match="memory guard"):
        B.factorize(w.op, w.row_tree, w.col_tree, w.recon)


@pytest.mark.parametrize("n", [1024, 4096])
def test_saturated_core_fit_newton_schulz(B, monkeypatch, n):
    """Config 3's saturated centre blocks (kv >= 64): the Newton-Schulz
    pseudo-inverse on batched DMMA GEMMs (k_corefit.cu) gives the core blocks
    of the one-sided Jacobi kernel (the reference's pinv_solve semantics,
    linalg.hpp:128-139): identical ranks, apply within 1e-11."""
    w = B.configs.build(3, n)
    a, la = B.factorize(w.op, w.row_tree, w.col_tree, w.recon)
    monkeypatch.setenv("BFLY_NO_BIG_CORE_FIT", "1")
    b, lb = B.factorize(w.op, w.row_tree, w.col_tree, w.recon)
    np.testing.assert_array_equal(a.rank_profile(), b.rank_profile())
    x = O.gaussian_matrix(n, 8, O.seed_mix(3, 3))
    e = rel_err(a.apply(x), b.apply(x))
    ta = la.phases[-1].seconds
    tb = lb.phases[-1].seconds
    print(f"config 3 n={n}: max rank {a.max_rank()}, centre level {ta*1e3:.1f} ms (Newton-Schulz) vs "
          f"{tb*1e3:.1f} ms (Jacobi), apply rel diff {e:.2e}")
    assert e < 1e-11


@pytest.mark.parametrize("case,vr", [("cfg4", 0), ("synth_real", 0), ("ragged", 0), ("cfg4", 3), ("cfg4_c64", 0)])
def test_structured_butterfly_products(tmp_path, case, vr):
    """Recompression (config 4): the butterfly black box multiplies a block
    only for the probes whose nonzero rows reach it
    (DevButterfly::apply_structured); the reference pads the probes and
    multiplies the zeros (reconstruct.hpp:72-85, operators.hpp:106-122).
    Three runs on the same seeds: padded (P), structured (S), structured with
    the basis projection answered by the black box (F, the default: the apply
    stops one level above the probes and multiplies G = B_new^H B_in, so the
    rest of its stages and the factorizer's projection chain disappear).  S
    skips exact zeros only, so it must reproduce P -- same ranks, same
    bookkeeping, apply outputs equal to rounding -- with fewer executed
    flops.  F associates the products differently: identical ranks and apply
    within 1e-12 at complex128; at complex64, where the ranks sit on the FP32
    noise floor, it may only lower them.  Also ragged leaves / varying ranks, a real butterfly and the
    rank-sharded schedule."""
    import os
    import subprocess
    import sys

    worker = os.path.join(os.path.dirname(__file__), "struct_worker.py")
    res = {}
    runs = [("P", {"BFLY_NO_STRUCT_APPLY": "1"}), ("S", {"BFLY_NO_LEAF_FUSE": "1"}), ("F", {})]
    if case == "cfg4" and vr == 0:
        # the projection is offered and declined: the factorizer multiplies again the plain way
        runs.append(("R", {"BFLY_DEBUG_REJECT_PROJ": "1"}))
    for tag, extra in runs:
        env = dict(os.environ)
        for k in ("BFLY_NO_STRUCT_APPLY", "BFLY_NO_LEAF_FUSE", "BFLY_DEBUG_REJECT_PROJ"):
            env.pop(k, None)
        env.update(extra)
        out = str(tmp_path / f"{tag}.npz")
        cmd = [sys.executable, worker, "--case", case, "--out", out] + (["--vr", str(vr)] if vr else [])
        subprocess.run(cmd, check=True, env=env, timeout=600)
        res[tag] = np.load(out)
    p, s, f = res["P"], res["S"], res["F"]
    if "R" in res:  # declined offers end in the structured products
        np.testing.assert_array_equal(res["R"]["profile"], s["profile"])
        np.testing.assert_array_equal(res["R"]["cols"], s["cols"])
        assert rel_err(res["R"]["yn"], s["yn"]) <= 1e-13 and float(res["R"]["flops"]) == float(s["flops"])
    assert bool(s["struct"]) and bool(f["struct"]) and not bool(p["struct"])
    c64 = case == "cfg4_c64"
    # structured = padded minus exact zeros
    np.testing.assert_array_equal(s["profile"], p["profile"])
    np.testing.assert_array_equal(s["cols"], p["cols"])
    tol = 1e-5 if c64 else 1e-13
    assert rel_err(s["yn"], p["yn"]) <= tol and rel_err(s["yh"], p["yh"]) <= tol
    assert float(s["flops"]) < float(p["flops"])
    # fused leaf projection (complex64: ranks, and with them the probe widths, follow the rounding noise)
    if c64:
        assert f["profile"].max() <= p["profile"].max() + 2
        assert rel_err(f["yn"], p["yn"]) <= 1e-4 and rel_err(f["yh"], p["yh"]) <= 1e-4
    else:
        np.testing.assert_array_equal(f["profile"], p["profile"])
        np.testing.assert_array_equal(f["cols"], p["cols"])
        assert rel_err(f["yn"], p["yn"]) <= 1e-12 and rel_err(f["yh"], p["yh"]) <= 1e-12
        assert float(f["flops"]) < float(s["flops"])
    print(f"{case} vr={vr}: S vs P apply {rel_err(s['yn'], p['yn']):.1e} / {rel_err(s['yh'], p['yh']):.1e}; "
          f"F vs P apply {rel_err(f['yn'], p['yn']):.1e} / {rel_err(f['yh'], p['yh']):.1e}; "
          f"flops P {float(p['flops']):.3e} S {float(s['flops']):.3e} F {float(f['flops']):.3e}; "
          f"ms P {float(p['seconds'])*1e3:.1f} S {float(s['seconds'])*1e3:.1f} F {float(f['seconds'])*1e3:.1f}")


@pytest.mark.parametrize("cfg_id,n,levels,over", [
    (0, 200, None, dict(tolerance=1e-3)),
    (0, 200, None, dict(tolerance=1e-9)),
    (0, 333, 2, {}),                                   # shallow tree: ragged leaves of ~83 points
    (2, 777, None, dict(oversampling=0)),
    (2, 777, None, dict(oversampling=6, rank_guess=1)),
    (1, 400, None, dict(rank_guess=64)),               # rank guess above the leaf size: capped rounds
    (2, 2048, 3, {}),                                  # 256-point leaves: large CPQR blocks
    (2, 130, 2, dict(tolerance=1e-12)),                # tolerance below what the leaves can resolve
])
def test_edge_configurations_match_oracle(B, oracle_threads, cfg_id, n, levels, over):
    """Corners of ReconstructionConfig and of the tree shape (core.hpp:166-196,
    reconstruct.hpp:352-399): loose / tight tolerances, no oversampling, a
    rank guess of 1 and one above the leaf size, shallow trees with large
    ragged leaves.  Identical rank profiles, bookkeeping (rounds, widths,
    rank_capped) and apply within 1e-10 of the oracle."""
    import dataclasses

    op_o, rt_o, ct_o, cfg = oracle_config(cfg_id, n, levels=levels)
    bf_o, log_o = O.factorize(op_o, rt_o, ct_o, dict(cfg, threads=oracle_threads, **over))
    w = B.configs.build(cfg_id, n, levels=levels)
    bf, log = B.factorize(w.op, w.row_tree, w.col_tree, dataclasses.replace(w.recon, **over))
    _compare(bf, log, bf_o, log_o, w.op.rows, w.op.cols)
