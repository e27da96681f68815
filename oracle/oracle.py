"""ctypes front end of the CPU ORACLE (test infrastructure only).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
reference legs import this module.  The product package never does.

Mirrors the reference API (/root/reference/proj/include/bfly/*.hpp) closely
enough that parity tests read like the reference's own Catch2 tests.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "_build", "libbfly_oracle.so")
_lib = None

OP_DENSE, OP_NUFFT, OP_PLATES, OP_CIRCLE, OP_COMPOSE, OP_BUTTERFLY = range(6)


class OracleError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"[{code}] {msg}")
        self.code = code


def build():
    subprocess.run(["make", "-s", "-C", _HERE], check=True)


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            build()
        L = C.CDLL(_LIB_PATH)
        p, i64, u64, dbl, i32 = C.c_void_p, C.c_int64, C.c_uint64, C.c_double, C.c_int
        sig = {
            "bo_last_error": (C.c_char_p, []),
            "bo_seed_mix": (u64, [u64, i32, p]),
            "bo_gaussian": (i32, [i64, i64, u64, i32, p]),
            "bo_tree_build": (p, [i32, i64, p, i32]),
            "bo_tree_from_table": (p, [i64, i32, p, p]),
            "bo_tree_free": (None, [p]),
            "bo_tree_table": (None, [p, p, p]),
            "bo_depth_for": (i32, [i64, i64]),
            "bo_cpqr_truncate": (i32, [i64, i64, p, i64, dbl, p, p, p, p]),
            "bo_pinv": (i32, [i64, i64, p, dbl, p]),
            "bo_householder_q": (i32, [i64, i64, p, p]),
            "bo_bf_free": (None, [p]),
            "bo_bf_validate": (i32, [p]),
            "bo_bf_nnz": (i64, [p]),
            "bo_bf_max_rank": (i64, [p]),
            "bo_bf_apply": (i32, [p, i32, p, i64, p]),
            "bo_bf_rank_profile": (i64, [p, p]),
            "bo_bf_serialize": (i64, [p, p]),
            "bo_bf_deserialize": (p, [p, i64]),
            "bo_bf_to_dense": (i32, [p, p]),
            "bo_op_dense": (p, [i64, i64, p, i32]),
            "bo_op_kernel": (p, [i32, i64, i64, p, p, dbl]),
            "bo_op_compose": (p, [p, p]),
            "bo_op_butterfly": (p, [p]),
            "bo_op_free": (None, [p]),
            "bo_op_rows": (i64, [p]),
            "bo_op_cols": (i64, [p]),
            "bo_op_apply": (i32, [p, i32, p, i64, p]),
            "bo_op_apply_adjoint": (i32, [p, p, i64, p]),
            "bo_op_counters": (None, [p, p, p]),
            "bo_op_reset_counters": (None, [p]),
            "bo_op_entry": (i32, [p, i64, i64, p]),
            "bo_set_threads": (None, [i32]),
            "bo_points_uniform": (None, [i64, u64, u64, dbl, dbl, p]),
            "bo_points_plate": (None, [i64, dbl, p]),
            "bo_points_half_circle": (None, [i64, i32, p]),
            "bo_synth_butterfly": (p, [i32, i64, i64, u64, i32, dbl]),
            "bo_cfg_default": (None, [p]),
            "bo_factorize": (i32, [p, p, p, p, p, p]),
            "bo_factorizer_new": (p, [p, p, p, p]),
            "bo_factorizer_leaf_row": (i32, [p]),
            "bo_factorizer_leaf_col": (i32, [p]),
            "bo_factorizer_transfer_w": (i32, [p, i32]),
            "bo_factorizer_transfer_r": (i32, [p, i32]),
            "bo_factorizer_complete": (i32, [p]),
            "bo_factorizer_take": (p, [p, p]),
            "bo_factorizer_free": (None, [p]),
            "bo_estimate_error": (i32, [p, p, i64, u64, p]),
            "bo_core_block": (i32, [i64, i64, p, i64, i64, p, i64, i64, p, i32, p]),
            "bo_probe_with": (i32, [p, p, i32, i64, p, i64, i64, i32, p]),
        }
        for name, (res, args) in sig.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


def _check(code):
    if code != 0:
        raise OracleError(code, lib().bo_last_error().decode())


def _ptr(a):
    return a.ctypes.data_as(C.c_void_p)


def _cmat(x, rows=None):
    a = np.asarray(x, dtype=np.complex128)
    if a.ndim == 1:
        a = a.reshape(-1, 1)
    return np.asfortranarray(a)


def set_threads(n):
    lib().bo_set_threads(int(n))


# ------------------------------------------------------------------ RNG ---
def seed_mix(seed, *words):
    w = np.array(words, dtype=np.uint64)
    return int(lib().bo_seed_mix(C.c_uint64(seed & (2**64 - 1)), len(words), _ptr(w) if len(w) else None))


def gaussian_matrix(rows, cols, seed, real=False):
    out = np.zeros((rows, cols), dtype=np.complex128, order="F") if rows > 0 and cols > 0 else np.zeros((1, 1), np.complex128)
    _check(lib().bo_gaussian(rows, cols, C.c_uint64(seed), int(real), _ptr(out)))
    return out.real.copy(order="F") if real else out


# --------------------------------------------------------------- linalg ---
def pivoted_qr_truncate(z, eps):
    z = _cmat(z)
    rows, cols = z.shape
    size = min(rows, cols)
    q = np.zeros((rows, max(size, 1)), np.complex128, order="F")
    k = C.c_int64(0)
    piv = np.zeros(max(cols, 1), np.int64)
    rd = np.zeros(max(size, 1), np.float64)
    _check(lib().bo_cpqr_truncate(rows, cols, _ptr(z), rows, eps, _ptr(q), C.byref(k), _ptr(piv), _ptr(rd)))
    return np.asfortranarray(q[:, : k.value]), k.value, piv[:cols], rd[:size]


def pinv_solve(m, tol=1e-12):
    m = _cmat(m)
    rows, cols = m.shape
    out = np.zeros((cols, rows), np.complex128, order="F")
    _check(lib().bo_pinv(rows, cols, _ptr(m), tol, _ptr(out)))
    return out


def householder_q(g):
    g = _cmat(g)
    q = np.zeros(g.shape, np.complex128, order="F")
    _check(lib().bo_householder_q(g.shape[0], g.shape[1], _ptr(g), _ptr(q)))
    return q


# ----------------------------------------------------------------- tree ---
class PartitionTree:
    def __init__(self, handle):
        self.h = handle
        self._load()

    def _load(self):
        # bo_tree layout: int levels; int64 n; ... -> use table export
        class _T(C.Structure):
            _fields_ = [("levels", C.c_int), ("n", C.c_int64), ("perm", C.c_void_p), ("rb", C.c_void_p)]

        t = _T.from_address(self.h)
        self.levels, self.n = t.levels, t.n
        total = sum((1 << l) + 1 for l in range(self.levels + 1))
        self.perm = np.zeros(self.n, np.int64)
        rb = np.zeros(total, np.int64)
        lib().bo_tree_table(self.h, _ptr(self.perm), _ptr(rb))
        self.ranges = []
        off = 0
        for l in range(self.levels + 1):
            c = (1 << l) + 1
            self.ranges.append(rb[off: off + c].copy())
            off += c
        self.range_flat = rb

    @staticmethod
    def build(points, levels, dim=None):
        pts = np.zeros((len(points), 3), np.float64)
        p = np.asarray(points, np.float64)
        if p.ndim == 1:
            p = p.reshape(-1, 1)
        pts[:, : p.shape[1]] = p
        d = dim or p.shape[1]
        h = lib().bo_tree_build(d, len(pts), _ptr(pts), levels)
        if not h:
            raise OracleError(1, lib().bo_last_error().decode())
        return PartitionTree(h)

    def node_range(self, l, j):
        return int(self.ranges[l][j]), int(self.ranges[l][j + 1])

    def __del__(self):
        try:
            lib().bo_tree_free(self.h)
        except Exception:
            pass


def depth_for(n, leaf):
    return lib().bo_depth_for(n, leaf)


# ------------------------------------------------------------ butterfly ---
class HybridButterfly:
    def __init__(self, handle, owned=True):
        self.h = handle
        self.owned = owned
        class _B(C.Structure):
            _fields_ = [("levels", C.c_int), ("center", C.c_int), ("rt", C.c_void_p), ("ct", C.c_void_p)]
        b = _B.from_address(handle)
        self.levels, self.center = b.levels, b.center
        self._rt, self._ct = b.rt, b.ct

    @property
    def rows(self):
        return C.c_int64.from_address(self._rt + 8).value

    @property
    def cols(self):
        return C.c_int64.from_address(self._ct + 8).value

    def apply(self, x, trans=0):
        x = _cmat(x)
        out_rows = self.rows if trans == 0 else self.cols
        y = np.zeros((out_rows, x.shape[1]), np.complex128, order="F")
        _check(lib().bo_bf_apply(self.h, trans, _ptr(x), x.shape[1], _ptr(y)))
        return y

    def apply_adjoint(self, y):
        return self.apply(y, 2)

    def apply_transpose(self, y):
        return self.apply(y, 1)

    def rank_profile(self):
        n = lib().bo_bf_rank_profile(self.h, None)
        out = np.zeros(n, np.int32)
        lib().bo_bf_rank_profile(self.h, _ptr(out))
        return out.reshape(self.levels + 2, 1 << self.levels)

    def nnz(self):
        return int(lib().bo_bf_nnz(self.h))

    def max_rank(self):
        return int(lib().bo_bf_max_rank(self.h))

    def serialize(self):
        n = lib().bo_bf_serialize(self.h, None)
        buf = np.zeros(n, np.uint8)
        lib().bo_bf_serialize(self.h, _ptr(buf))
        return buf.tobytes()

    @staticmethod
    def deserialize(data: bytes):
        buf = np.frombuffer(data, np.uint8).copy()
        h = lib().bo_bf_deserialize(_ptr(buf), len(buf))
        if not h:
            raise OracleError(4, lib().bo_last_error().decode())
        return HybridButterfly(h)

    def to_dense(self):
        out = np.zeros((self.rows, self.cols), np.complex128, order="F")
        _check(lib().bo_bf_to_dense(self.h, _ptr(out)))
        return out

    def validate(self):
        _check(lib().bo_bf_validate(self.h))

    def release(self):
        self.owned = False
        return self.h

    def __del__(self):
        if getattr(self, "owned", False):
            try:
                lib().bo_bf_free(self.h)
            except Exception:
                pass


def synth_butterfly(levels, rank, seed, leaf=8, real=False, perturb=0.0):
    h = lib().bo_synth_butterfly(levels, leaf, rank, C.c_uint64(seed), int(real), perturb)
    if not h:
        raise OracleError(1, lib().bo_last_error().decode())
    return HybridButterfly(h)


# ------------------------------------------------------------ operators ---
class Operator:
    def __init__(self, handle, keep=()):
        self.h = handle
        self._keep = keep

    @property
    def rows(self):
        return int(lib().bo_op_rows(self.h))

    @property
    def cols(self):
        return int(lib().bo_op_cols(self.h))

    def apply(self, x):
        x = _cmat(x)
        y = np.zeros((self.rows, x.shape[1]), np.complex128, order="F")
        _check(lib().bo_op_apply(self.h, 0, _ptr(x), x.shape[1], _ptr(y)))
        return y

    def apply_transpose(self, x):
        x = _cmat(x)
        y = np.zeros((self.cols, x.shape[1]), np.complex128, order="F")
        _check(lib().bo_op_apply(self.h, 1, _ptr(x), x.shape[1], _ptr(y)))
        return y

    def apply_adjoint(self, x):
        x = _cmat(x)
        y = np.zeros((self.cols, x.shape[1]), np.complex128, order="F")
        _check(lib().bo_op_apply_adjoint(self.h, _ptr(x), x.shape[1], _ptr(y)))
        return y

    def counters(self):
        f, t = C.c_int64(0), C.c_int64(0)
        lib().bo_op_counters(self.h, C.byref(f), C.byref(t))
        return f.value, t.value

    def entry(self, i, j):
        out = np.zeros(1, np.complex128)
        _check(lib().bo_op_entry(self.h, i, j, _ptr(out)))
        return out[0]

    def release(self):
        h, self.h = self.h, None
        return h

    def __del__(self):
        if getattr(self, "h", None):
            try:
                lib().bo_op_free(self.h)
            except Exception:
                pass


def dense_operator(a, real=False):
    a = _cmat(a)
    return Operator(lib().bo_op_dense(a.shape[0], a.shape[1], _ptr(a), int(real)))


def kernel_operator(kind, tgt, src, kappa=0.0):
    t = np.ascontiguousarray(tgt, np.float64)
    s = np.ascontiguousarray(src, np.float64)
    return Operator(lib().bo_op_kernel(kind, len(t), len(s), _ptr(t), _ptr(s), kappa))


def compose_operator(f2: Operator, f1: Operator):
    return Operator(lib().bo_op_compose(f2.release(), f1.release()))


def butterfly_operator(bf: HybridButterfly):
    return Operator(lib().bo_op_butterfly(bf.release()))


# -------------------------------------------------------- reconstruction ---
class _Cfg(C.Structure):
    _fields_ = [
        ("tolerance", C.c_double), ("oversampling", C.c_int64), ("rank_guess", C.c_int64),
        ("levels", C.c_int), ("center", C.c_int), ("seed", C.c_uint64), ("hard_cap", C.c_int64),
        ("threads", C.c_int), ("literal_transpose_core", C.c_int),
    ]


class _Phase(C.Structure):
    _fields_ = [("name", C.c_char * 32), ("forward_columns", C.c_int64), ("transpose_columns", C.c_int64),
                ("seconds", C.c_double), ("rounds", C.c_int), ("probe_width", C.c_int64),
                ("rank_margin", C.c_double)]


class _Log(C.Structure):
    _fields_ = [("nphases", C.c_int), ("phases", _Phase * 64), ("peak_probe_bytes", C.c_uint64),
                ("peak_concurrent_probes", C.c_int64), ("rank_capped", C.c_int), ("total_seconds", C.c_double)]


def _mk_cfg(cfg: dict):
    c = _Cfg()
    lib().bo_cfg_default(C.byref(c))
    for k, v in cfg.items():
        setattr(c, k, v)
    return c


def _log_dict(lg: _Log):
    phases = []
    for i in range(lg.nphases):
        p = lg.phases[i]
        phases.append(dict(name=p.name.decode(), forward_columns=p.forward_columns,
                           transpose_columns=p.transpose_columns, seconds=p.seconds,
                           rounds=p.rounds, probe_width=p.probe_width, rank_margin=p.rank_margin))
    return dict(phases=phases, peak_probe_bytes=lg.peak_probe_bytes,
                peak_concurrent_probes=lg.peak_concurrent_probes, rank_capped=bool(lg.rank_capped),
                total_seconds=lg.total_seconds)


def factorize(op: Operator, row_tree: PartitionTree, col_tree: PartitionTree, cfg: dict):
    c = _mk_cfg(cfg)
    out = C.c_void_p(0)
    lg = _Log()
    _check(lib().bo_factorize(op.h, row_tree.h, col_tree.h, C.byref(c), C.byref(out), C.byref(lg)))
    return HybridButterfly(out.value), _log_dict(lg)


class Factorizer:
    """Phase-stepping API (reconstruct.hpp:175-321)."""

    def __init__(self, op, row_tree, col_tree, cfg):
        c = _mk_cfg(cfg)
        self.h = lib().bo_factorizer_new(op.h, row_tree.h, col_tree.h, C.byref(c))
        if not self.h:
            raise OracleError(1, lib().bo_last_error().decode())

    def leaf_row_bases(self):
        _check(lib().bo_factorizer_leaf_row(self.h))

    def leaf_col_bases(self):
        _check(lib().bo_factorizer_leaf_col(self.h))

    def transfer_level_w(self, l):
        _check(lib().bo_factorizer_transfer_w(self.h, l))

    def transfer_level_r(self, l):
        _check(lib().bo_factorizer_transfer_r(self.h, l))

    def complete(self):
        return bool(lib().bo_factorizer_complete(self.h))

    def __del__(self):
        try:
            lib().bo_factorizer_free(self.h)
        except Exception:
            pass


def estimate_error(op: Operator, bf: HybridButterfly, k=16, seed=0):
    e = C.c_double(0)
    _check(lib().bo_estimate_error(op.h, bf.h, k, C.c_uint64(seed), C.byref(e)))
    return e.value


def core_block(k_omega, u, v_coeff, literal=False):
    """core_block (reconstruct.hpp:125-138)."""
    z, u, cf = _cmat(k_omega), _cmat(u), _cmat(v_coeff)
    out = np.zeros((u.shape[1], cf.shape[0]), np.complex128, order="F") if u.shape[1] * cf.shape[0] else np.zeros(1, np.complex128)
    _check(lib().bo_core_block(z.shape[0], z.shape[1], _ptr(z), u.shape[0], u.shape[1], _ptr(u), cf.shape[0],
                               cf.shape[1], _ptr(cf), int(literal), _ptr(out)))
    return out.reshape(u.shape[1], cf.shape[0], order="F")


def probe_with(op: Operator, tree: PartitionTree, level, node, core, forward=True):
    """probe_with (reconstruct.hpp:72-85)."""
    c = _cmat(core)
    rows = op.rows if forward else op.cols
    out = np.zeros((rows, c.shape[1]), np.complex128, order="F")
    _check(lib().bo_probe_with(op.h, tree.h, level, node, _ptr(c), c.shape[0], c.shape[1], int(forward), _ptr(out)))
    return out
