"""The BASELINE.json configurations, built through the product API.

Builder decisions (recorded in DESIGN.md "Configs"): points are generated,
a tree is built, the points are re-indexed into tree order and the tree is
rebuilt, so both permutations are the identity (tests/test_tree.cpp:86-98
pins that property of the bisection).  Uniform points come from the
splitmix stream seed_mix(op_seed, tag); probe seed 0; oversampling 2.

  0  NUFFT        n=4096,  leaf 32, r0 16, tol 1e-6
  1  3D plates    n=16384 (128x128), leaf 32, r0 16, tol 1e-6, k = 2 pi / (10 h)
  2  half circles n=65536, leaf 32, r0 4,  tol 1e-6, k = 2 n / 10
  3  F2 * F1      n=65536, leaf 32, r0 16, tol 1e-5 (operator seeds 1, 2)
  4  recompress   n=262144 (L=12, leaf 64, rank 32), r0 16, tol 1e-6,
                  perturbation 1e-8, input seed 0
Every config accepts a smaller n for the parity tests.
"""
from __future__ import annotations

import dataclasses
import math

import numpy as np

from . import api
from ._native import lib

FULL_N = {0: 4096, 1: 16384, 2: 65536, 3: 65536, 4: 262144}


def _vp(a):
    import ctypes as C

    return a.ctypes.data_as(C.c_void_p)


def points_uniform(n, seed, tag, lo, hi):
    out = np.zeros((n, 3), np.float64)
    lib().bfly_points_uniform(n, seed, tag, lo, hi, _vp(out))
    return out


def points_plate(side, z):
    out = np.zeros((side * side, 3), np.float64)
    lib().bfly_points_plate(side, z, _vp(out))
    return out


def points_half_circle(n, upper):
    out = np.zeros((n, 3), np.float64)
    lib().bfly_points_half_circle(n, 1 if upper else 0, _vp(out))
    return out


def tree_order(points, levels, dim):
    """Re-index points into tree order; returns (ordered points, identity tree)."""
    t = api.PartitionTree.build(points[:, :dim], levels, dim)
    pts = np.ascontiguousarray(points[t.perm])
    t2 = api.PartitionTree.build(pts[:, :dim], levels, dim)
    assert (t2.perm == np.arange(len(pts))).all()
    return pts, t2


@dataclasses.dataclass
class Workload:
    cfg_id: int
    n: int
    op: object
    row_tree: object
    col_tree: object
    recon: api.ReconstructionConfig
    name: str
    meta: dict


def nufft_points(n, op_seed):
    x = points_uniform(n, op_seed, 1, 0.0, 1.0)
    xi = points_uniform(n, op_seed, 2, -n / 2.0, n / 2.0)
    return x, xi


def build(cfg_id: int, n: int | None = None, scalar=api.COMPLEX128, ctx=None, seed: int = 0,
          levels: int | None = None) -> Workload:
    """``levels`` overrides the tree depth (default: depth_for(n, leaf)),
    like the reference CLI's --L (tools/bfly_cli.cpp:351)."""
    n = n or FULL_N[cfg_id]

    def depth(nn, leaf):
        return levels if levels else api.PartitionTree.depth_for(nn, leaf)
    if cfg_id == 0:
        L = depth(n, 32)
        x, xi = nufft_points(n, 0)
        x, rt = tree_order(x, L, 1)
        xi, ct = tree_order(xi, L, 1)
        op = api.NufftOperator(x, xi, scalar=scalar, ctx=ctx)
        rc = api.ReconstructionConfig(tolerance=1e-6, rank_guess=16, levels=L, seed=seed)
        return Workload(0, n, op, rt, ct, rc, f"nufft1d_n{n}", dict(leaf=32))
    if cfg_id == 1:
        side = int(round(math.sqrt(n)))
        assert side * side == n, "plates need a square point count"
        L = depth(n, 32)
        h = 1.0 / side
        kappa = 2.0 * math.pi / (10.0 * h)
        t, rt = tree_order(points_plate(side, 0.0), L, 3)
        s, ct = tree_order(points_plate(side, 2.0), L, 3)
        op = api.HelmholtzPlatesOperator(t, s, kappa, scalar=scalar, ctx=ctx)
        rc = api.ReconstructionConfig(tolerance=1e-6, rank_guess=16, levels=L, seed=seed)
        return Workload(1, n, op, rt, ct, rc, f"helmholtz_plates_n{n}", dict(leaf=32, kappa=kappa))
    if cfg_id == 2:
        L = depth(n, 32)
        kappa = 2.0 * n / 10.0
        t, rt = tree_order(points_half_circle(n, True), L, 2)
        s, ct = tree_order(points_half_circle(n, False), L, 2)
        op = api.HelmholtzCircleOperator(t, s, kappa, scalar=scalar, ctx=ctx)
        rc = api.ReconstructionConfig(tolerance=1e-6, rank_guess=4, levels=L, seed=seed)
        return Workload(2, n, op, rt, ct, rc, f"helmholtz_circle_n{n}", dict(leaf=32, kappa=kappa))
    if cfg_id == 3:
        L = depth(n, 32)
        x1, xi1 = nufft_points(n, 1)
        x2, xi2 = nufft_points(n, 2)
        x2, rt = tree_order(x2, L, 1)      # rows of A = F2's targets
        xi1, ct = tree_order(xi1, L, 1)    # cols of A = F1's sources
        f1 = api.NufftOperator(x1, xi1, scalar=scalar, ctx=ctx)
        f2 = api.NufftOperator(x2, xi2, scalar=scalar, ctx=ctx)
        op = api.CompositionOperator(f2, f1, ctx=ctx)
        rc = api.ReconstructionConfig(tolerance=1e-5, rank_guess=16, levels=L, seed=seed)
        return Workload(3, n, op, rt, ct, rc, f"nufft_composition_n{n}", dict(leaf=32))
    if cfg_id == 4:
        leaf, rank = 64, 32
        L = depth(n, leaf)
        bf = api.synth_butterfly(L, rank, 0, leaf=leaf, scalar=scalar, perturb=1e-8, ctx=ctx)
        rt = api.PartitionTree.build(np.arange(n, dtype=np.float64), L)
        op = api.ButterflyOperator(bf, ctx=ctx)
        rc = api.ReconstructionConfig(tolerance=1e-6, rank_guess=16, levels=L, seed=seed)
        return Workload(4, n, op, rt, rt, rc, f"recompress_n{n}", dict(leaf=leaf, rank=rank, perturb=1e-8))
    raise ValueError(f"unknown config {cfg_id}")
