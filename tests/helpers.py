"""Oracle-side builders of the BASELINE configs (same recipe as
paper_2002_03400_b200/configs.py, through the CPU oracle's own generators)."""
import math

import numpy as np

import oracle as O


def _uniform(n, seed, tag, lo, hi):
    out = np.zeros((n, 3))
    O.lib().bo_points_uniform(n, seed, tag, lo, hi, O._ptr(out))
    return out


def _plate(side, z):
    out = np.zeros((side * side, 3))
    O.lib().bo_points_plate(side, z, O._ptr(out))
    return out


def _half_circle(n, upper):
    out = np.zeros((n, 3))
    O.lib().bo_points_half_circle(n, 1 if upper else 0, O._ptr(out))
    return out


def _tree_order(pts, L, dim):
    t = O.PartitionTree.build(pts[:, :dim], L, dim)
    p = np.ascontiguousarray(pts[t.perm])
    t2 = O.PartitionTree.build(p[:, :dim], L, dim)
    assert (t2.perm == np.arange(len(p))).all()
    return p, t2


def oracle_config(cfg_id, n, seed=0, levels=None):
    """-> (op, row_tree, col_tree, cfg dict); ``levels`` overrides the tree
    depth of configs 0-2 (like configs.build)"""
    if cfg_id == 0:
        L = levels or O.depth_for(n, 32)
        x, rt = _tree_order(_uniform(n, 0, 1, 0.0, 1.0), L, 1)
        xi, ct = _tree_order(_uniform(n, 0, 2, -n / 2.0, n / 2.0), L, 1)
        op = O.kernel_operator(O.OP_NUFFT, x, xi)
        return op, rt, ct, dict(levels=L, tolerance=1e-6, rank_guess=16, oversampling=2, seed=seed)
    if cfg_id == 1:
        side = int(round(math.sqrt(n)))
        L = levels or O.depth_for(n, 32)
        kappa = 2.0 * math.pi / (10.0 * (1.0 / side))
        t, rt = _tree_order(_plate(side, 0.0), L, 3)
        s, ct = _tree_order(_plate(side, 2.0), L, 3)
        op = O.kernel_operator(O.OP_PLATES, t, s, kappa)
        return op, rt, ct, dict(levels=L, tolerance=1e-6, rank_guess=16, oversampling=2, seed=seed)
    if cfg_id == 2:
        L = levels or O.depth_for(n, 32)
        t, rt = _tree_order(_half_circle(n, True), L, 2)
        s, ct = _tree_order(_half_circle(n, False), L, 2)
        op = O.kernel_operator(O.OP_CIRCLE, t, s, 2.0 * n / 10.0)
        return op, rt, ct, dict(levels=L, tolerance=1e-6, rank_guess=4, oversampling=2, seed=seed)
    if cfg_id == 3:
        L = O.depth_for(n, 32)
        x1, xi1 = _uniform(n, 1, 1, 0.0, 1.0), _uniform(n, 1, 2, -n / 2.0, n / 2.0)
        x2, xi2 = _uniform(n, 2, 1, 0.0, 1.0), _uniform(n, 2, 2, -n / 2.0, n / 2.0)
        x2, rt = _tree_order(x2, L, 1)
        xi1, ct = _tree_order(xi1, L, 1)
        f1 = O.kernel_operator(O.OP_NUFFT, x1, xi1)
        f2 = O.kernel_operator(O.OP_NUFFT, x2, xi2)
        op = O.compose_operator(f2, f1)
        return op, rt, ct, dict(levels=L, tolerance=1e-5, rank_guess=16, oversampling=2, seed=seed)
    if cfg_id == 4:
        L = O.depth_for(n, 64)
        bf = O.synth_butterfly(L, 32, 0, leaf=64, perturb=1e-8)
        rt = O.PartitionTree.build(np.arange(n, dtype=float), L)
        op = O.butterfly_operator(bf)
        return op, rt, rt, dict(levels=L, tolerance=1e-6, rank_guess=16, oversampling=2, seed=seed)
    raise ValueError(cfg_id)


def rel_err(a, b):
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


def oracle_points(cfg_id, n):
    """Tree-ordered (targets, sources, kernel kind, kappa) of a kernel config,
    through the oracle's generators (configs 0-2)."""
    if cfg_id == 0:
        L = O.depth_for(n, 32)
        x, _ = _tree_order(_uniform(n, 0, 1, 0.0, 1.0), L, 1)
        xi, _ = _tree_order(_uniform(n, 0, 2, -n / 2.0, n / 2.0), L, 1)
        return x, xi, O.OP_NUFFT, 0.0
    if cfg_id == 1:
        side = int(round(math.sqrt(n)))
        L = O.depth_for(n, 32)
        t, _ = _tree_order(_plate(side, 0.0), L, 3)
        s, _ = _tree_order(_plate(side, 2.0), L, 3)
        return t, s, O.OP_PLATES, 2.0 * math.pi / (10.0 * (1.0 / side))
    if cfg_id == 2:
        L = O.depth_for(n, 32)
        t, _ = _tree_order(_half_circle(n, True), L, 2)
        s, _ = _tree_order(_half_circle(n, False), L, 2)
        return t, s, O.OP_CIRCLE, 2.0 * n / 10.0
    raise ValueError(cfg_id)
