"""Python front end of the B200 butterfly construction library.

Mirrors the reference C++ API (/root/reference/proj/include/bfly/):
``PartitionTree`` (tree.hpp), ``BlackBoxOperator`` and its subclasses
(operators.hpp), ``ReconstructionConfig`` / ``Factorizer`` / ``factorize`` /
``estimate_error`` (reconstruct.hpp), ``HybridButterfly`` (butterfly.hpp) and
the ``.bfh`` container (serialize.hpp).  Every call goes through the C ABI
(include/bfly_b200.h) into sm_100a kernels; host numpy buffers are copied in
and out inside the call, torch CUDA tensors are used in place.
"""
from __future__ import annotations

import atexit
import ctypes as C
from dataclasses import dataclass
import dataclasses
from typing import Optional

import numpy as np

from ._native import (APPLY_FN, APPLY_RANGE_FN, BflyError, ConditioningError, Cfg, CudaError, DimensionError,
                      FormatError, Log, NcclError, PreconditionError, SequencingError, check, lib)

COMPLEX128, COMPLEX64, REAL64 = 0, 1, 2
_NP = {COMPLEX128: np.complex128, COMPLEX64: np.complex64, REAL64: np.float64}
N, T, H = 0, 1, 2
OP_DENSE, OP_NUFFT, OP_PLATES, OP_CIRCLE, OP_COMPOSE, OP_BUTTERFLY, OP_CALLBACK = range(7)


def _vp(a):
    return a.ctypes.data_as(C.c_void_p)


# Native handles are released by __del__ while the interpreter runs; at exit
# the process teardown reclaims them instead (finalizers of objects kept alive
# until shutdown -- e.g. by a stored traceback -- run in no particular order,
# so a butterfly could otherwise be destroyed after its context).
_FINALIZING = [False]
atexit.register(lambda: _FINALIZING.__setitem__(0, True))


def _live() -> bool:
    return not _FINALIZING[0]


# ------------------------------------------------------------------ context
class Context:
    """One GPU: stream, memory pool, optional NCCL communicator."""

    _default = {}

    def __init__(self, device: int = 0):
        h = C.c_void_p()
        check(lib().bfly_ctx_create(device, C.byref(h)))
        self.h = h
        self.device = device

    @classmethod
    def default(cls, device: int = 0) -> "Context":
        if device not in cls._default:
            cls._default[device] = Context(device)
        return cls._default[device]

    @property
    def launches(self) -> int:
        return int(lib().bfly_ctx_launches(self.h))

    @property
    def stream(self) -> int:
        return int(lib().bfly_ctx_stream(self.h) or 0)

    def synchronize(self):
        check(lib().bfly_ctx_synchronize(self.h))

    def profile(self, enable: int = 1):
        """Per-kernel CUDA-event timing on the library stream (1 on, 0 off, -1 off+clear)."""
        check(lib().bfly_ctx_profile(self.h, enable))

    def profile_report(self) -> dict:
        import json

        n = lib().bfly_ctx_profile_report(self.h, None, 0)
        buf = C.create_string_buffer(int(n))
        lib().bfly_ctx_profile_report(self.h, buf, n)
        return json.loads(buf.value.decode())

    def set_comm(self, rank: int, world: int, unique_id: bytes):
        buf = (C.c_uint8 * 128).from_buffer_copy(unique_id.ljust(128, b"\0")[:128])
        check(lib().bfly_ctx_set_comm(self.h, rank, world, buf))

    def set_host_comm(self, group=None):
        """Join the host-staged transport over an initialized torch.distributed
        process group (gloo): same sharded schedule as set_comm, every exchange
        staged through pinned host memory (ranks may share one GPU)."""
        from .hostcomm import TorchHostComm

        hc = TorchHostComm(group)
        check(lib().bfly_ctx_set_host_comm(self.h, hc.rank, hc.world, C.byref(hc.fns)))
        self._host_comm = hc  # the library holds its function pointers
        return hc

    def comm_info(self):
        """(rank, world, transport) with transport 'none' | 'nccl' | 'host'."""
        r, w, t = C.c_int(), C.c_int(), C.c_int()
        check(lib().bfly_ctx_comm_info(self.h, C.byref(r), C.byref(w), C.byref(t)))
        return r.value, w.value, ("none", "nccl", "host")[t.value]

    @staticmethod
    def unique_id() -> bytes:
        buf = (C.c_uint8 * 128)()
        check(lib().bfly_comm_unique_id(buf))
        return bytes(buf)

    def __del__(self):
        try:
            if not _live():
                return
            if getattr(self, "h", None):
                lib().bfly_ctx_destroy(self.h)
        except Exception:
            pass


def _ctx(ctx):
    return ctx if ctx is not None else Context.default()


# --------------------------------------------------------------------- trees

class PartitionTree:
    """Complete bisection tree (tree.hpp:66-216)."""

    def __init__(self, handle):
        self.h = handle
        n, lv = C.c_int64(), C.c_int()
        check(lib().bfly_tree_info(handle, C.byref(n), C.byref(lv)))
        self.n, self._levels = n.value, lv.value
        total = sum((1 << l) + 1 for l in range(self._levels + 1))
        self.perm = np.zeros(self.n, np.int64)
        flat = np.zeros(total, np.int64)
        check(lib().bfly_tree_table(handle, _vp(self.perm), _vp(flat)))
        self.ranges, off = [], 0
        for l in range(self._levels + 1):
            self.ranges.append(flat[off: off + (1 << l) + 1].copy())
            off += (1 << l) + 1
        self.flat_ranges = flat

    @staticmethod
    def build(points, levels: int, dim: Optional[int] = None) -> "PartitionTree":
        p = np.asarray(points, np.float64)
        if p.ndim == 1:
            p = p.reshape(-1, 1)
        pts = np.zeros((p.shape[0], 3), np.float64)
        pts[:, : p.shape[1]] = p
        h = C.c_void_p()
        check(lib().bfly_tree_build(dim or p.shape[1], pts.shape[0], _vp(pts), levels, C.byref(h)))
        return PartitionTree(h)

    @staticmethod
    def from_table(perm, ranges) -> "PartitionTree":
        perm = np.ascontiguousarray(perm, np.int64)
        flat = np.ascontiguousarray(np.concatenate([np.asarray(r, np.int64) for r in ranges]))
        h = C.c_void_p()
        check(lib().bfly_tree_from_table(len(perm), len(ranges) - 1, _vp(perm), _vp(flat), C.byref(h)))
        return PartitionTree(h)

    @staticmethod
    def depth_for(n: int, leaf_cap: int) -> int:
        d = lib().bfly_depth_for(n, leaf_cap)
        if d < 0:
            raise PreconditionError("depth_for: leaf_cap >= 1 required")
        return d

    def levels(self) -> int:
        return self._levels

    def size(self) -> int:
        return self.n

    def node_range(self, level: int, pos: int):
        return int(self.ranges[level][pos]), int(self.ranges[level][pos + 1])

    def node_size(self, level: int, pos: int) -> int:
        b, e = self.node_range(level, pos)
        return e - b

    def to_original(self, slot: int) -> int:
        return int(self.perm[slot])

    def __del__(self):
        try:
            if not _live():
                return
            lib().bfly_tree_destroy(self.h)
        except Exception:
            pass


# ------------------------------------------------------------------ buffers
def _is_torch_cuda(x) -> bool:
    return hasattr(x, "is_cuda") and bool(getattr(x, "is_cuda"))


def _host_in(x, scalar):
    a = np.asarray(x, dtype=_NP[scalar])
    if a.ndim == 1:
        a = a.reshape(-1, 1)
    return np.asfortranarray(a)


class _Applicable:
    """Shared N / T / H application logic (host numpy or torch CUDA tensors)."""

    scalar: int

    def _rows_in(self, trans):
        return self.cols if trans == N else self.rows

    def _rows_out(self, trans):
        return self.rows if trans == N else self.cols

    def _call(self, trans, x, out=None):
        if _is_torch_cuda(x):
            import torch

            # the device kernels read and write the object's own scalar type
            want = {COMPLEX128: torch.complex128, COMPLEX64: torch.complex64, REAL64: torch.float64}[self.scalar]
            if x.dim() == 1:
                x = x.reshape(-1, 1)
            if x.dim() != 2:
                raise DimensionError(f"apply: X must be 1-D or 2-D, got {x.dim()}-D")
            if x.shape[0] != self._rows_in(trans):
                raise DimensionError(f"apply: X row count {x.shape[0]} != {self._rows_in(trans)}")
            if x.dtype != want:
                if x.is_complex() and not want.is_complex:
                    raise PreconditionError(f"apply: complex input for a real ({want}) object")
                x = x.to(want)
            k, rows_out = x.shape[1], self._rows_out(trans)

            def ld_of(t):  # column-major leading dimension (a single column may report any stride)
                return max(t.stride(1), t.shape[0]) if t.shape[1] == 1 else t.stride(1)

            def colmajor(t):
                return t.stride(0) == 1 and ld_of(t) >= t.shape[0]

            # column-major (ld >= rows): a transposed contiguous tensor
            xt = x if colmajor(x) else x.t().contiguous().t()
            if out is not None:
                if out.dtype != want or tuple(out.shape) != (rows_out, k) or not colmajor(out) or not out.is_cuda:
                    raise DimensionError(f"apply: out must be a column-major {want} CUDA tensor of shape "
                                         f"({rows_out}, {k})")
                y = out
            else:
                y = torch.empty((k, rows_out), dtype=want, device=x.device).t()
            torch.cuda.current_stream().synchronize()
            check(self._apply_fn(trans, C.c_void_p(xt.data_ptr()), ld_of(xt), C.c_void_p(y.data_ptr()), ld_of(y), k, 1))
            self._ctx().synchronize()
            return y
        a = _host_in(x, self.scalar)
        if a.shape[0] != self._rows_in(trans):
            raise DimensionError(f"apply: X row count {a.shape[0]} != {self._rows_in(trans)}")
        y = np.zeros((self._rows_out(trans), a.shape[1]), dtype=_NP[self.scalar], order="F")
        check(self._apply_fn(trans, _vp(a), a.shape[0], _vp(y), y.shape[0], a.shape[1], 0))
        return y


# ---------------------------------------------------------------- operators
class BlackBoxOperator(_Applicable):
    """BlackBoxOperator<Scalar> (operators.hpp:17-56) living on the GPU."""

    kind = -1

    def __init__(self, handle, ctx, scalar):
        self.h = handle
        self.ctx = ctx
        self.scalar = scalar
        m, n = C.c_int64(), C.c_int64()
        check(lib().bfly_op_info(handle, C.byref(m), C.byref(n), None, None))
        self.rows, self.cols = m.value, n.value

    def _ctx(self):
        return self.ctx

    def _apply_fn(self, trans, x, ldx, y, ldy, k, dev):
        return lib().bfly_op_apply(self.h, trans, x, ldx, y, ldy, k, dev)

    def apply(self, x, out=None):
        return self._call(N, x, out)

    def apply_transpose(self, y, out=None):
        return self._call(T, y, out)

    def apply_adjoint(self, y, out=None):
        return self._call(H, y, out)

    def _counters(self):
        f, t = C.c_int64(), C.c_int64()
        check(lib().bfly_op_counters(self.h, C.byref(f), C.byref(t)))
        return f.value, t.value

    def forward_columns(self) -> int:
        return self._counters()[0]

    def transpose_columns(self) -> int:
        return self._counters()[1]

    def total_columns(self) -> int:
        return sum(self._counters())

    def reset_counters(self):
        check(lib().bfly_op_reset_counters(self.h))

    def _release(self):
        h, self.h = self.h, None
        return h

    def __del__(self):
        try:
            if not _live():
                return
            if getattr(self, "h", None):
                lib().bfly_op_destroy(self.h)
        except Exception:
            pass


def apply_adjoint(op: BlackBoxOperator, y):
    """K^H Y through the black box (operators.hpp:59-66)."""
    return op.apply_adjoint(y)


def _pts3(p):
    p = np.asarray(p, np.float64)
    if p.ndim == 1:
        p = p.reshape(-1, 1)
    out = np.zeros((p.shape[0], 3), np.float64)
    out[:, : p.shape[1]] = p
    return np.ascontiguousarray(out)


class KernelOperator(BlackBoxOperator):
    def __init__(self, kind, targets, sources, wavenumber=0.0, scalar=COMPLEX128, ctx=None):
        ctx = _ctx(ctx)
        t, s = _pts3(targets), _pts3(sources)
        h = C.c_void_p()
        check(lib().bfly_op_kernel(ctx.h, kind, len(t), len(s), _vp(t), _vp(s), float(wavenumber), scalar,
                                   C.byref(h)))
        self.kind = kind
        self.targets, self.sources, self.wavenumber = t, s, wavenumber
        super().__init__(h, ctx, scalar)


class NufftOperator(KernelOperator):
    """A_ij = exp(2 pi i x_i xi_j)  (BASELINE config 0)."""

    def __init__(self, x, xi, scalar=COMPLEX128, ctx=None):
        super().__init__(OP_NUFFT, x, xi, 0.0, scalar, ctx)


class HelmholtzPlatesOperator(KernelOperator):
    """exp(i k r) / (4 pi r) between two plates  (BASELINE config 1)."""

    def __init__(self, targets, sources, wavenumber, scalar=COMPLEX128, ctx=None):
        super().__init__(OP_PLATES, targets, sources, wavenumber, scalar, ctx)


class HelmholtzCircleOperator(KernelOperator):
    """exp(i k r) / r between two half circles  (BASELINE config 2)."""

    def __init__(self, targets, sources, wavenumber, scalar=COMPLEX128, ctx=None):
        super().__init__(OP_CIRCLE, targets, sources, wavenumber, scalar, ctx)


class CompositionOperator(BlackBoxOperator):
    """A = F2 F1 applied as two sequential products (BASELINE config 3).
    Takes ownership of both factors."""

    kind = OP_COMPOSE

    def __init__(self, f2: BlackBoxOperator, f1: BlackBoxOperator, ctx=None):
        ctx = _ctx(ctx)
        h = C.c_void_p()
        scalar = f1.scalar
        check(lib().bfly_op_compose(ctx.h, f2._release(), f1._release(), C.byref(h)))
        super().__init__(h, ctx, scalar)


class DenseOperator(BlackBoxOperator):
    """DenseOperator (operators.hpp:68-85)."""

    kind = OP_DENSE

    def __init__(self, a, scalar=None, ctx=None):
        ctx = _ctx(ctx)
        a = np.asarray(a)
        if scalar is None:
            scalar = REAL64 if np.isrealobj(a) else COMPLEX128
        arr = np.asfortranarray(a.astype(_NP[scalar]))
        h = C.c_void_p()
        check(lib().bfly_op_dense(ctx.h, arr.shape[0], arr.shape[1], _vp(arr), scalar, C.byref(h)))
        self.matrix = arr
        super().__init__(h, ctx, scalar)


class ButterflyOperator(BlackBoxOperator):
    """ButterflyOperator (operators.hpp:105-122); takes ownership of bf."""

    kind = OP_BUTTERFLY

    def __init__(self, bf: "HybridButterfly", ctx=None):
        ctx = _ctx(ctx)
        h = C.c_void_p()
        scalar = bf.scalar
        check(lib().bfly_op_butterfly(ctx.h, bf._release(), C.byref(h)))
        super().__init__(h, ctx, scalar)


class CallbackOperator(BlackBoxOperator):
    """User black box: fn(trans, x_ptr, ldx, y_ptr, ldy, k, stream) -> int on
    device buffers (trans 0 = A x, 1 = A^T y).  ranged=True: fn(trans, x_ptr,
    ldx, y_ptr, ldy, k, nz_begin, nz_end, stream), called once per structured
    probe with its nonzero input rows [nz_begin, nz_end) (bfly_apply_range_fn)."""

    kind = OP_CALLBACK

    def __init__(self, m, n, fn, scalar=COMPLEX128, ctx=None, ranged=False):
        ctx = _ctx(ctx)

        if ranged:
            def tramp(user, trans, x, ldx, y, ldy, k, b, e, stream):
                try:
                    return int(fn(trans, x, ldx, y, ldy, k, b, e, stream) or 0)
                except Exception:  # surfaced as a failed black-box call
                    import traceback

                    traceback.print_exc()
                    return 5

            self._cb = APPLY_RANGE_FN(tramp)
            register = lib().bfly_op_callback_ranged
        else:
            def tramp(user, trans, x, ldx, y, ldy, k, stream):
                try:
                    return int(fn(trans, x, ldx, y, ldy, k, stream) or 0)
                except Exception:  # surfaced as a failed black-box call
                    return 5

            self._cb = APPLY_FN(tramp)
            register = lib().bfly_op_callback
        h = C.c_void_p()
        check(register(ctx.h, m, n, scalar, self._cb, None, C.byref(h)))
        super().__init__(h, ctx, scalar)


# ------------------------------------------------------------ reconstruction
@dataclasses.dataclass
class ReconstructionConfig:
    """reconstruct.hpp:10-36 (+ max_batch_probes: probes per black-box launch)."""

    tolerance: float = 1e-6
    oversampling: int = 2
    rank_guess: int = 4
    levels: int = 4
    center: int = -1
    seed: int = 0
    hard_cap: int = -1
    threads: int = 1
    literal_transpose_core: bool = False
    max_batch_probes: int = 0
    virtual_ranks: int = 0

    def center_level(self) -> int:
        return self.levels // 2 if self.center < 0 else self.center

    def _c(self) -> Cfg:
        c = Cfg()
        lib().bfly_cfg_default(C.byref(c))
        for f in dataclasses.fields(self):
            v = getattr(self, f.name)
            setattr(c, f.name, int(v) if f.name != "tolerance" else float(v))
        return c


@dataclasses.dataclass
class PhaseStat:
    name: str
    forward_columns: int
    transpose_columns: int
    seconds: float
    rounds: int
    probe_width: int
    # CPQR cut margin (bfly_phase.rank_margin): min over the phase's blocks of
    # min(|R_{k-1}|/thr - 1, 1 - |R_k|/thr), thr = 0.25 tol |R_00|; inf: none
    rank_margin: float = float("inf")


@dataclasses.dataclass
class FactorizationLog:
    """FactorizationLog (reconstruct.hpp:95-120) + algorithmic work counters."""

    phases: list
    peak_probe_bytes: int
    peak_concurrent_probes: int
    rank_capped: bool
    total_seconds: float
    flops: float
    kernel_evals: float
    products_recomputed: bool = False  # the K2 range check sent the factorization to the FP64 path

    @staticmethod
    def _from(lg: Log) -> "FactorizationLog":
        ph = [PhaseStat(p.name.decode(), p.forward_columns, p.transpose_columns, p.seconds, p.rounds, p.probe_width,
                        p.rank_margin)
              for p in lg.phases[: lg.nphases]]
        return FactorizationLog(ph, lg.peak_probe_bytes, lg.peak_concurrent_probes, bool(lg.rank_capped),
                                lg.total_seconds, lg.flops, lg.kernel_evals, bool(lg.products_recomputed))

    def forward_columns(self) -> int:
        return sum(p.forward_columns for p in self.phases)

    def transpose_columns(self) -> int:
        return sum(p.transpose_columns for p in self.phases)

    def total_columns(self) -> int:
        return self.forward_columns() + self.transpose_columns()

    def phase(self, name: str) -> Optional[PhaseStat]:
        for p in self.phases:
            if p.name == name:
                return p
        return None


class HybridButterfly(_Applicable):
    """HybridButterfly on the GPU (butterfly.hpp:20-387)."""

    def __init__(self, handle, ctx):
        self.h = handle
        self.ctx = ctx
        lv, ce, sc = C.c_int(), C.c_int(), C.c_int()
        m, n, nnz, mr = C.c_int64(), C.c_int64(), C.c_int64(), C.c_int64()
        check(lib().bfly_bf_info(handle, C.byref(lv), C.byref(ce), C.byref(m), C.byref(n), C.byref(nnz),
                                 C.byref(mr), C.byref(sc)))
        self.levels, self.center, self.rows, self.cols = lv.value, ce.value, m.value, n.value
        self.scalar = sc.value
        self._nnz, self._max_rank = nnz.value, mr.value

    def _ctx(self):
        return self.ctx

    def _apply_fn(self, trans, x, ldx, y, ldy, k, dev):
        return lib().bfly_apply(self.h, trans, x, ldx, y, ldy, k, dev)

    def apply(self, x, out=None):
        return self._call(N, x, out)

    def apply_adjoint(self, y, out=None):
        return self._call(H, y, out)

    def apply_transpose(self, y, out=None):
        return self._call(T, y, out)

    def apply_layout(self, x, spec: "LayoutSpec", trans: int = N):
        """The apply executed over a process layout (inc/layout.hpp:139-261).
        With a communicator on the context (one process per GPU) the
        coefficient blocks move by NCCL send/recv; otherwise
        ``spec.processes`` virtual processes run in turn on this GPU.  Returns
        (y, measured CommCostReport, {"max_recv": ..., "total_recv": ...} --
        scalars per column actually moved)."""
        if spec.levels != self.levels:
            raise DimensionError("apply_layout: spec level count does not match the butterfly")
        rep = (C.c_double * 6)()

        def fn(trans_, x_, ldx, y_, ldy, k, dev):
            return lib().bfly_apply_layout(self.h, trans_, spec.kind_id, spec.processes, x_, ldx, y_, ldy, k, dev,
                                           rep)

        self._apply_fn = fn  # instance override for this call only
        try:
            y = self._call(trans, x)
        finally:
            del self._apply_fn
        measured = CommCostReport(rep[0], int(rep[1]), rep[2], int(rep[3]))
        return y, measured, {"max_recv": rep[4], "total_recv": rep[5]}

    def nnz(self) -> int:
        return self._nnz

    def max_rank(self) -> int:
        return self._max_rank

    def apply_flops_per_column(self) -> int:
        return 2 * self._nnz

    def rank_profile(self) -> np.ndarray:
        """(L+2) x 2^L: u ranks for levels center..L, then v ranks for 0..center."""
        n = lib().bfly_rank_profile(self.h, None)
        out = np.zeros(n, np.int32)
        lib().bfly_rank_profile(self.h, _vp(out))
        return out.reshape(self.levels + 2, 1 << self.levels)

    def serialized_size(self) -> int:
        n = lib().bfly_serialize(self.h, None)
        if n < 0:
            check(6)
        return int(n)

    def serialize(self, out=None):
        """.bfh container bytes (reference format, serialize.hpp:103-127).

        Factor blocks are packed into the file layout on the GPU and read back
        with one device-to-host copy.  ``out``: optional writable buffer of at
        least ``serialized_size()`` bytes (e.g. a reused pinned host buffer --
        filling fresh pageable memory costs more than the export itself);
        returns a memoryview of the written bytes.  Without ``out`` a new
        bytearray is returned."""
        n = self.serialized_size()
        buf = bytearray(n) if out is None else out
        view = (C.c_uint8 * n).from_buffer(buf)
        rc = lib().bfly_serialize(self.h, view)
        del view
        if rc < 0:
            check(6)
        return buf if out is None else memoryview(buf).cast("B")[:n]

    @staticmethod
    def deserialize(data: bytes, scalar=COMPLEX128, ctx=None) -> "HybridButterfly":
        ctx = _ctx(ctx)
        buf = np.frombuffer(data, np.uint8).copy()
        h = C.c_void_p()
        check(lib().bfly_deserialize(ctx.h, _vp(buf), len(buf), scalar, C.byref(h)))
        return HybridButterfly(h, ctx)

    def convert(self, scalar) -> "HybridButterfly":
        h = C.c_void_p()
        check(lib().bfly_bf_convert(self.h, scalar, C.byref(h)))
        return HybridButterfly(h, self.ctx)

    def save(self, path: str):
        with open(path, "wb") as f:
            f.write(self.serialize())

    @staticmethod
    def load(path: str, scalar=COMPLEX128, ctx=None) -> "HybridButterfly":
        with open(path, "rb") as f:
            return HybridButterfly.deserialize(f.read(), scalar, ctx)

    def _release(self):
        h, self.h = self.h, None
        return h

    def __del__(self):
        try:
            if not _live():
                return
            if getattr(self, "h", None):
                lib().bfly_bf_destroy(self.h)
        except Exception:
            pass


def factorize(op: BlackBoxOperator, row_tree: PartitionTree, col_tree: PartitionTree,
              cfg: ReconstructionConfig):
    """factorize (reconstruct.hpp:412-419) -> (HybridButterfly, FactorizationLog)."""
    h = C.c_void_p()
    lg = Log()
    check(lib().bfly_factorize(op.ctx.h, op.h, row_tree.h, col_tree.h, C.byref(cfg._c()), C.byref(h), C.byref(lg)))
    return HybridButterfly(h, op.ctx), FactorizationLog._from(lg)


class Factorizer:
    """Phase-stepping API (reconstruct.hpp:145-321)."""

    def __init__(self, op: BlackBoxOperator, row_tree: PartitionTree, col_tree: PartitionTree,
                 cfg: ReconstructionConfig):
        h = C.c_void_p()
        check(lib().bfly_factorizer_create(op.ctx.h, op.h, row_tree.h, col_tree.h, C.byref(cfg._c()), C.byref(h)))
        self.h, self.ctx, self._op = h, op.ctx, op

    def leaf_row_bases(self):
        check(lib().bfly_factorizer_leaf_row_bases(self.h))

    def leaf_col_bases(self):
        check(lib().bfly_factorizer_leaf_col_bases(self.h))

    def transfer_level_w(self, l: int):
        check(lib().bfly_factorizer_transfer_level_w(self.h, l))

    def transfer_level_r(self, l: int):
        check(lib().bfly_factorizer_transfer_level_r(self.h, l))

    def complete(self) -> bool:
        return bool(lib().bfly_factorizer_complete(self.h))

    def take(self):
        h = C.c_void_p()
        lg = Log()
        check(lib().bfly_factorizer_take(self.h, C.byref(h), C.byref(lg)))
        return HybridButterfly(h, self.ctx), FactorizationLog._from(lg)

    def __del__(self):
        try:
            if not _live():
                return
            lib().bfly_factorizer_destroy(self.h)
        except Exception:
            pass


# ---------------------------------------------------------------- layouts
LAYOUT_KINDS = ("column", "row", "hybrid")


def layout_name(kind: str) -> str:
    return kind


def layout_from_name(name: str) -> str:
    """layout_from_name (layout.hpp:20-25)."""
    if name not in LAYOUT_KINDS:
        raise PreconditionError("unknown layout kind: " + str(name))
    return name


@dataclass
class LayoutSpec:
    """LayoutSpec (layout.hpp:27-49): kind, L, constant model rank r, p."""

    kind: str = "hybrid"
    levels: int = 4
    rank: int = 8
    processes: int = 1

    @property
    def kind_id(self) -> int:
        return LAYOUT_KINDS.index(layout_from_name(self.kind))

    def log_p(self) -> int:
        g = 0
        while (1 << (g + 1)) <= self.processes:
            g += 1
        return g


@dataclass
class CommCostReport:
    """CommCostReport (layout.hpp:52-66), scalars per input column."""

    exchange_volume: float = 0.0
    exchange_msgs: int = 0
    alltoall_volume: float = 0.0
    alltoall_msgs: int = 0

    def model_time(self, alpha: float, beta: float) -> float:
        return alpha * (self.exchange_msgs + self.alltoall_msgs) + beta * (self.exchange_volume + self.alltoall_volume)


def comm_cost(spec: LayoutSpec) -> CommCostReport:
    """Closed-form model (layout.hpp:70-88); invalid specs raise PreconditionError."""
    out = (C.c_double * 4)()
    check(lib().bfly_comm_cost(spec.kind_id, spec.levels, spec.rank, spec.processes, out))
    return CommCostReport(out[0], int(out[1]), out[2], int(out[3]))


@dataclass
class OwnershipMap:
    """OwnershipMap (layout.hpp:113-136): owners by flat block index."""

    processes: int
    levels: int
    center: int
    u_leaf: np.ndarray
    v_leaf: np.ndarray
    r_owner: np.ndarray  # [l - center][block]
    w_owner: np.ndarray  # [l - 1][block]
    b_owner: np.ndarray

    def r_at(self, level, tau, nu):
        return int(self.r_owner[level - self.center][tau * (1 << (self.levels - level)) + nu])

    def w_at(self, level, tau, nu):
        return int(self.w_owner[level - 1][tau * (1 << (self.levels - level)) + nu])

    def b_at(self, tau, nu):
        return int(self.b_owner[tau * (1 << (self.levels - self.center)) + nu])


def assign_ownership(bf, spec: LayoutSpec) -> OwnershipMap:
    """assign_ownership (layout.hpp:139-188).  ``bf`` is a HybridButterfly or
    a (levels, center) pair (the map depends on nothing else)."""
    levels, center = (bf.levels, bf.center) if hasattr(bf, "levels") else bf
    if spec.levels != levels:
        raise DimensionError("assign_ownership: spec level count does not match the butterfly")
    n = lib().bfly_layout_owners(spec.kind_id, levels, center, spec.processes, None)
    if n < 0:
        check(int(-n))
    out = np.zeros(n, np.int32)
    lib().bfly_layout_owners(spec.kind_id, levels, center, spec.processes, _vp(out))
    nb = 1 << levels
    o = out.reshape(-1, nb)
    return OwnershipMap(spec.processes, levels, center, o[0].copy(), o[1].copy(), o[2:2 + levels - center].copy(),
                        o[2 + levels - center:2 + levels].copy(), o[2 + levels].copy())


def estimate_error(op: BlackBoxOperator, bf: HybridButterfly, k: int = 16, seed: int = 0) -> float:
    """estimate_error (reconstruct.hpp:423-434)."""
    e = C.c_double()
    check(lib().bfly_estimate_error(op.h, bf.h, k, seed, C.byref(e)))
    return e.value


def residuals(op: BlackBoxOperator, bf: HybridButterfly) -> dict:
    """Level-wise residual sums against a dense copy of ``op`` (desk scale),
    reconstruct.hpp:443-503: ``u`` (l = L..l_m, u_side_residual), ``v``
    (l = 0..l_m, v_side_residual), ``center`` (center_residual) and
    ``knorm2`` = ||K||_F^2.  The operator is densified on the GPU."""
    u = np.zeros(bf.levels - bf.center + 1)
    v = np.zeros(bf.center + 1)
    cen, kn = C.c_double(), C.c_double()
    check(lib().bfly_residuals(op.h, bf.h, _vp(u), _vp(v), C.byref(cen), C.byref(kn)))
    return {"u": u, "v": v, "center": cen.value, "knorm2": kn.value}


def synth_butterfly(levels: int, rank: int, seed: int, leaf: int = 8, scalar=COMPLEX128, perturb: float = 0.0,
                    ctx=None) -> HybridButterfly:
    """synth_butterfly (operators.hpp:131-178), generalised to leaf b."""
    ctx = _ctx(ctx)
    h = C.c_void_p()
    check(lib().bfly_synth_butterfly(ctx.h, levels, leaf, rank, seed, scalar, perturb, C.byref(h)))
    return HybridButterfly(h, ctx)


# --------------------------------------------------------------- dense bits
def seed_mix(seed: int, *words) -> int:
    w = np.array(words, np.uint64)
    return int(lib().bfly_seed_mix(seed, len(w), _vp(w) if len(w) else None))


def gaussian_matrix(rows: int, cols: int, seed: int, scalar=COMPLEX128, ctx=None) -> np.ndarray:
    ctx = _ctx(ctx)
    out = np.zeros((rows, cols), dtype=_NP[scalar], order="F") if rows > 0 and cols > 0 else np.zeros(1)
    check(lib().bfly_gaussian(ctx.h, rows, cols, seed, scalar, _vp(out)))
    return out


def pivoted_qr_truncate(z, eps: float, ctx=None):
    """Truncated column-pivoted QR on the device (linalg.hpp:62-80) -> Q."""
    ctx = _ctx(ctx)
    z = np.asfortranarray(np.asarray(z, np.complex128))
    q = np.zeros((z.shape[0], max(1, min(z.shape))), np.complex128, order="F")
    k = C.c_int64()
    check(lib().bfly_cpqr_truncate(ctx.h, z.shape[0], z.shape[1], _vp(z), eps, _vp(q), C.byref(k)))
    return np.asfortranarray(q[:, : k.value])


def pinv_solve(m, tol: float = 1e-12, ctx=None):
    """Pseudo-inverse on the device (linalg.hpp:128-139)."""
    ctx = _ctx(ctx)
    m = np.asfortranarray(np.asarray(m, np.complex128))
    out = np.zeros((m.shape[1], m.shape[0]), np.complex128, order="F")
    check(lib().bfly_pinv(ctx.h, m.shape[0], m.shape[1], _vp(m), tol, _vp(out)))
    return out


__all__ = [
    "residuals", "BflyError", "PreconditionError", "DimensionError", "SequencingError", "FormatError", "ConditioningError",
    "CudaError", "NcclError", "Context", "PartitionTree", "BlackBoxOperator", "apply_adjoint", "NufftOperator",
    "HelmholtzPlatesOperator", "HelmholtzCircleOperator", "CompositionOperator", "DenseOperator",
    "ButterflyOperator", "CallbackOperator", "KernelOperator", "ReconstructionConfig", "PhaseStat",
    "FactorizationLog", "HybridButterfly", "factorize", "Factorizer", "estimate_error", "synth_butterfly",
    "seed_mix", "gaussian_matrix", "pivoted_qr_truncate", "pinv_solve", "COMPLEX128", "COMPLEX64", "REAL64",
]
