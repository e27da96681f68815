"""ctypes front end of oracle/_ref/libbfly_ref.so: the REFERENCE implementation
(its headers compiled unmodified against oracle/ref/eigen_shim).  Test
infrastructure only (tests/, bench.py --impl reference)."""
import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB = os.path.join(_HERE, "_ref", "libbfly_ref.so")
_lib = None


def available():
    return os.path.exists(LIB)


def lib():
    global _lib
    if _lib is None:
        L = C.CDLL(LIB)
        p, i64, u64, i32, dbl = C.c_void_p, C.c_int64, C.c_uint64, C.c_int, C.c_double
        pp = C.POINTER(C.c_void_p)
        sig = {
            "ref_last_error": (C.c_char_p, []),
            "ref_set_threads": (None, [i32]),
            "ref_op_kernel": (i32, [i32, i64, i64, p, p, dbl, i32, i32, pp]),
            "ref_op_compose": (i32, [i64, p, p, p, p, i32, pp]),
            "ref_op_butterfly": (i32, [p, i64, pp]),
            "ref_op_synth": (i32, [i32, i64, u64, pp]),
            "ref_op_free": (None, [p]),
            "ref_factorize": (i32, [p, dbl, i64, i64, i32, u64, i32, pp]),
            "ref_rank_profile": (i64, [p, p]),
            "ref_apply": (i32, [p, i32, p, i64, p]),
            "ref_log": (i32, [p, p, p, p, p]),
            "ref_estimate_error": (dbl, [p, p, i64, u64]),
            "ref_phase_seconds": (i32, [p, p, p]),
            "ref_serialize": (i64, [p, p]),
            "ref_bf_free": (None, [p]),
            "ref_probe_sample": (dbl, [p, i32, i32, i64, u64]),
            "ref_seed_mix": (u64, [u64, i32, p]),
            "ref_gaussian": (i32, [i32, i64, i64, u64, p]),
            "ref_cpqr": (i64, [i64, i64, p, dbl, p]),
            "ref_residuals": (i32, [p, p, p, p, p, p]),
            "ref_comm_cost": (i32, [i32, i32, i64, i64, p]),
            "ref_layout_synth": (i32, [i32, i64, u64, i32, i64, p, p]),
            "ref_layout_bf": (i32, [p, i32, i64, p, p]),
        }
        for k, (r, a) in sig.items():
            f = getattr(L, k)
            f.restype, f.argtypes = r, a
        _lib = L
    return _lib


def _vp(a):
    return a.ctypes.data_as(C.c_void_p)


def _check(rc):
    if rc != 0:
        raise RuntimeError(f"[{rc}] {lib().ref_last_error().decode()}")


class RefOp:
    def __init__(self, h, rows, cols):
        self.h, self.rows, self.cols = h, rows, cols

    def __del__(self):
        try:
            lib().ref_op_free(self.h)
        except Exception:
            pass


def kernel_op(kind, tgt, src, kappa, dim, L):
    t, s = np.ascontiguousarray(tgt, np.float64), np.ascontiguousarray(src, np.float64)
    h = C.c_void_p()
    _check(lib().ref_op_kernel(kind, len(t), len(s), _vp(t), _vp(s), kappa, dim, L, C.byref(h)))
    return RefOp(h, len(t), len(s))


def compose_op(n, x2, xi2, x1, xi1, L):
    arrs = [np.ascontiguousarray(a, np.float64) for a in (x2, xi2, x1, xi1)]
    h = C.c_void_p()
    _check(lib().ref_op_compose(n, *[_vp(a) for a in arrs], L, C.byref(h)))
    return RefOp(h, n, n)


def butterfly_op(bfh: bytes):
    buf = np.frombuffer(bytes(bfh), np.uint8).copy()
    h = C.c_void_p()
    _check(lib().ref_op_butterfly(_vp(buf), len(buf), C.byref(h)))
    n = int(np.frombuffer(bytes(bfh)[17:25], np.uint64)[0])  # rows: magic, version, tag, L, lm precede
    return RefOp(h, n, n)


def synth_op(levels, rank, seed):
    h = C.c_void_p()
    _check(lib().ref_op_synth(levels, rank, seed, C.byref(h)))
    n = (1 << levels) * 8
    return RefOp(h, n, n)


class RefButterfly:
    def __init__(self, h, op):
        self.h, self.op = h, op

    def rank_profile(self, levels):
        n = lib().ref_rank_profile(self.h, None)
        out = np.zeros(n, np.int32)
        lib().ref_rank_profile(self.h, _vp(out))
        return out.reshape(levels + 2, 1 << levels)

    def apply(self, x, trans=0):
        x = np.asfortranarray(x, np.complex128)
        rows = self.op.cols if trans else self.op.rows
        y = np.zeros((rows, x.shape[1]), np.complex128, order="F")
        _check(lib().ref_apply(self.h, trans, _vp(x), x.shape[1], _vp(y)))
        return y

    def log(self):
        cols = np.zeros(128, np.int64)
        rounds = np.zeros(64, np.int32)
        widths = np.zeros(64, np.int64)
        tot = C.c_double()
        n = lib().ref_log(self.h, _vp(cols), _vp(rounds), _vp(widths), C.byref(tot))
        return [(int(cols[2 * i]), int(cols[2 * i + 1]), int(rounds[i]), int(widths[i])) for i in range(n)], tot.value

    def phase_seconds(self):
        """[(name, seconds)] of the reference's FactorizationLog (reconstruct.hpp:87-120)."""
        n = lib().ref_phase_seconds(self.h, None, None)
        sec = np.zeros(n)
        names = np.zeros(32 * n, np.uint8)
        lib().ref_phase_seconds(self.h, _vp(sec), _vp(names))
        return [(bytes(names[32 * i: 32 * i + 32]).split(b"\0")[0].decode(), float(sec[i])) for i in range(n)]

    def estimate_error(self, k=16, seed=0):
        """estimate_error(op, bf, k, seed) of the reference (reconstruct.hpp:423-434)."""
        return float(lib().ref_estimate_error(self.op.h, self.h, k, seed))

    def residuals(self, levels, center):
        """(u[l=L..lm], v[l=0..lm], center, ||K||^2) of the reference."""
        u = np.zeros(levels - center + 1)
        v = np.zeros(center + 1)
        cen, kn = C.c_double(), C.c_double()
        _check(lib().ref_residuals(self.op.h, self.h, _vp(u), _vp(v), C.byref(cen), C.byref(kn)))
        return u, v, cen.value, kn.value

    def layout(self, levels, kind, p):
        """(simulated_parallel_apply tallies[4], owners[(L+3) 2^L]) (layout.hpp:139-261)."""
        out = np.zeros(4)
        own = np.zeros((levels + 3) << levels, np.int32)
        _check(lib().ref_layout_bf(self.h, kind, p, _vp(out), _vp(own)))
        return out, own

    def serialize(self):
        n = lib().ref_serialize(self.h, None)
        buf = np.zeros(n, np.uint8)
        lib().ref_serialize(self.h, _vp(buf))
        return buf.tobytes()

    def __del__(self):
        try:
            lib().ref_bf_free(self.h)
        except Exception:
            pass


def factorize(op: RefOp, tol, r0, L, seed=0, p=2, threads=1):
    h = C.c_void_p()
    _check(lib().ref_factorize(op.h, tol, p, r0, L, seed, threads, C.byref(h)))
    return RefButterfly(h, op)


def seed_mix(seed, *words):
    w = np.array(words, dtype=np.uint64)
    return int(lib().ref_seed_mix(seed, len(words), _vp(w) if len(words) else None))


def gaussian_matrix(rows, cols, seed, complex_=True):
    out = np.zeros((cols, rows), dtype=np.complex128 if complex_ else np.float64)
    _check(lib().ref_gaussian(1 if complex_ else 0, rows, cols, seed, _vp(out)))
    return out.T  # column-major storage -> (rows, cols) view


def pivoted_qr_truncate(w, eps):
    """returns (rank, Q); rank -2 marks the reference's zero_input case"""
    w = np.asarray(w, dtype=np.complex128)
    rows, cols = w.shape
    buf = np.asfortranarray(w)
    q = np.zeros((min(rows, cols), rows), dtype=np.complex128)
    rank = lib().ref_cpqr(rows, cols, _vp(buf), eps, _vp(q))
    if rank == -1:
        raise RuntimeError(lib().ref_last_error().decode())
    k = max(rank, 0)
    return rank, q[:k].T.copy()


def comm_cost(kind, levels, rank, p):
    """comm_cost (layout.hpp:70-88) -> [exchange_volume, exchange_msgs, alltoall_volume, alltoall_msgs]."""
    out = np.zeros(4)
    _check(lib().ref_comm_cost(kind, levels, rank, p, _vp(out)))
    return out


def layout_synth(levels, rank, seed, kind, p):
    """The reference's synthetic butterfly through assign_ownership + simulated_parallel_apply."""
    out = np.zeros(4)
    own = np.zeros((levels + 3) << levels, np.int32)
    _check(lib().ref_layout_synth(levels, rank, seed, kind, p, _vp(out), _vp(own)))
    return out, own
