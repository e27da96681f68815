#!/usr/bin/env python
"""Benchmark: adaptive butterfly construction on BASELINE config 2.

Workload (BASELINE.json metric "butterfly construction sec & GFLOP/s at
n=65536 complex128; apply GB/s"): the weak-admissibility 2D Helmholtz
operator exp(ikr)/r between two half circles, n = 65536 points each,
complex128, tol 1e-6, leaf 32 (L = 11), r0 = 4, evaluated on the fly.
A step = one full factorize() (both adaptive leaf phases, 5 W levels,
6 R levels + core fit).  GFLOP/s = algorithmic flops (DESIGN.md 8d:
black-box contraction + chain projections + QR + core fit; kernel-entry
evaluations are not counted as flops) / construction time.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl reference]

N > 1 runs under torchrun: one process per GPU.  Default (--mode shard): ONE
construction whose level probes are sharded across the ranks with an NCCL
all-gather of every level's new blocks (strong scaling).  --mode replica: every
rank factorizes its own copy (weak scaling).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "butterfly construction GFLOP/s at n=65536 complex128 (config 2)"
FP64_PEAK_TFLOPS = 36.99  # measured DMMA m8n8k4 f64 on this pool (profiles/r01_fp64_peaks.txt)
INT8_PEAK_TOPS = 4248.7  # measured tcgen05 kind::i8 M128 N256 from shared memory (profiles/r01_tc_i8.txt)
# dram__bytes_read.sum + dram__bytes_write.sum of one K2 launch (the 9th of a config-2 construction: 32
# probe segments x 32 columns, profiles/r02_k2_ncu_s2.txt): 56.0 MB read + 1018.5 MB write (= the
# 1.07 GB product it writes); its algorithmic traffic (points + probes in, product out) is 1.11 GB
K2_DRAM_BYTES_PER_LAUNCH = 1074533056
# the same capture: FP64 pipe 40.3 % + int8 tensor pipe 33.2 % busy; on B200 both run on one shared
# datapath (sm__pipe_shared_cycles_active 73.5 %), the utilisation that bounds K2
K2_PIPES = {"fp64": 0.403, "tensor_int8": 0.332, "shared_datapath": 0.735}
CFG_ID = 2


def _hbm_peak():
    """measured copy bandwidth (MEASURED_PEAKS.json, driver-written), else the recipe's fallback"""
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return float(json.load(f)["hbm_gbs"])
    except Exception:
        return 6650.0


HBM_PEAK_GBS = _hbm_peak()


def _env_rank():
    return int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)), int(os.environ.get("LOCAL_RANK", 0))


# ------------------------------------------------------------ CPU baseline
def cpu_sample(n=65536, probes=8, width=32, threads=None):
    """Bounded sample of the same workload on the CPU: the adjoint black-box
    products of `probes` level-5 row probes (|T_tau| = n/32 rows, `width`
    columns, all n output points) -- the operation that carries >90% of the
    construction's flops.  Runs the REFERENCE code path (oracle/_ref:
    reference headers compiled unmodified against the Eigen-API shim;
    probe_with -> apply_adjoint -> conj(apply_transpose(conj))) when it was
    built, else the C oracle port of the same path."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import oracle as O
    import refpy as RP
    from helpers import _half_circle, _tree_order, oracle_config

    threads = threads or os.cpu_count() or 1
    level = 5
    flops = 8.0 * n * (n >> level) * width * probes
    if RP.available():
        RP.lib().ref_set_threads(threads)
        L = O.depth_for(n, 32)
        t, _ = _tree_order(_half_circle(n, True), L, 2)
        s, _ = _tree_order(_half_circle(n, False), L, 2)
        op = RP.kernel_op(3, t, s, 2.0 * n / 10.0, 2, L)
        dt = RP.lib().ref_probe_sample(op.h, level, probes, width, 0)
        kind, what = "reference", "reference probe_with (oracle/_ref)"
    else:
        O.set_threads(threads)
        op, rt, ct, cfg = oracle_config(CFG_ID, n)
        t0 = time.perf_counter()
        for tau in range(probes):
            b, e = rt.node_range(level, tau)
            core = O.gaussian_matrix(e - b, width, O.seed_mix(0, 3, level, tau))
            O.probe_with(op, rt, level, tau, core, forward=False)
        dt = time.perf_counter() - t0
        kind, what = "port", "C oracle port"
    return flops / dt / 1e9, dt, threads, kind, (
        f"adjoint black-box products of {probes} W-level-{level} row probes of config 2 "
        f"(n={n}, {n >> level} rows x {width} cols each) via the {what}, {threads} threads")


# algorithmic flops of one config-2 construction, counted by the library's log; the
# reference factorization has the identical rank profile and bookkeeping (tests/test_full_parity.py),
# hence the same count
CFG2_FLOPS = 14371885543744.0
SAMPLE_SCOPE = ("a bounded SAMPLE of the construction, not a whole factorize(): the black-box products of "
                "W-level-5 row probes (the operation carrying > 90 % of the construction's flops), through the "
                "reference's own probe_with + operator; the whole reference factorize() is under full_construction")


def full_reference_construction():
    """The reference's own full config-2 factorize() (oracle/_ref, all host threads), timed once on the
    GPU box's host by tests/golden/make_fullsize_golden.py (FactorizationLog.total_seconds,
    reconstruct.hpp:309-314) -- reported beside the sampled rate, not re-run per bench step (~3 min)."""
    try:
        import numpy as np

        d = np.load(os.path.join(ROOT, "tests", "golden", "full_cfg2.npz"))
        sec = float(d["total_seconds"])
        return {"seconds": round(sec, 2), "GFLOP/s": round(CFG2_FLOPS / sec / 1e9, 2), "threads": int(d["threads"]),
                "cpu": str(d["cpu_model"]), "producer": str(d["producer"]),
                "phases_s": {str(k): round(float(v), 2) for k, v in zip(d["phase_names"], d["phase_seconds"])},
                "source": "tests/golden/full_cfg2.npz (tests/golden/make_fullsize_golden.py on the GPU box host)"}
    except Exception as e:  # fixture missing: say so
        return {"unavailable": str(e)}


def run_reference(args):
    rank, world, _ = _env_rank()
    if rank != 0:
        return 0
    vals = []
    for i in range(args.warmup + args.steps):
        v, dt, threads, kind, sample = cpu_sample(probes=args.ref_probes)
        if i >= args.warmup:
            vals.append((v, dt))
    value = statistics.median(v for v, _ in vals)
    ms = statistics.mean(dt for _, dt in vals) * 1e3
    line = {
        "impl": "reference", "metric": METRIC, "value": round(value, 3), "unit": "GFLOP/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms, 3), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "complex128", "data": "synthetic",
        "config": {"workload": "config2_helmholtz_circle_n65536", "n": 65536, "sample": sample},
        "cpu_baseline": {"value": round(value, 3), "unit": "GFLOP/s", "cores": threads, "kind": kind,
                         "sample": sample, "scope": SAMPLE_SCOPE,
                         "full_construction": full_reference_construction()},
        "e2e": {"value": round(value, 3), "unit": "GFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# -------------------------------------------------------------- clocks
class ClockSampler:
    def __init__(self, index):
        self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
        q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        try:
            self.p = subprocess.Popen(["nvidia-smi", f"--id={index}", f"--query-gpu={q}", "--format=csv,noheader,nounits",
                                       "-lms", "200"], stdout=self.f, stderr=subprocess.DEVNULL)
        except Exception:
            self.p = None

    def stop(self):
        if self.p is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.p.terminate()
        self.p.wait()
        self.f.flush()
        self.f.seek(0)
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in self.f.read().splitlines():
            parts = [x.strip() for x in line.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1]))
                mx = float(parts[2])
            except ValueError:
                continue
            for nm, v in zip(names, parts[5:9]):
                if v.lower() == "active":
                    reasons.add(nm)
        os.unlink(self.f.name)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


# ------------------------------------------------------------------ ours
def run_ours(args):
    import numpy as np
    import torch

    import paper_2002_03400_b200 as B

    rank, world, local = _env_rank()
    ndev = torch.cuda.device_count()
    transport = args.transport
    if transport == "auto":
        transport = "nccl" if world <= ndev else "host"
    if transport == "nccl" and world > ndev:
        raise SystemExit(f"bench: {world} ranks need {world} GPUs for NCCL, {ndev} visible (use --transport host)")
    local = local % ndev
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist

        if transport == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group("gloo")
    red_dev = "cuda" if transport == "nccl" else "cpu"

    def barrier():
        if dist is not None:
            dist.barrier()
        torch.cuda.synchronize()

    def allreduce(v, op):
        t = torch.tensor([v], dtype=torch.float64, device=red_dev)
        if dist is not None:
            dist.all_reduce(t, op=dist.ReduceOp.MAX if op == "max" else dist.ReduceOp.SUM)
        return t.item()

    ctx = B.Context(local)
    sharded = world > 1 and args.mode == "shard"
    if sharded:
        if transport == "nccl":
            uid = [B.Context.unique_id() if rank == 0 else None]
            dist.broadcast_object_list(uid, src=0)
            ctx.set_comm(rank, world, uid[0])
        else:
            ctx.set_host_comm()
    stream = torch.cuda.ExternalStream(ctx.stream)
    w = B.configs.build(CFG_ID, args.size or None, ctx=ctx)
    op, rt, ct, rc = w.op, w.row_tree, w.col_tree, w.recon
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")  # 256 MB > L2

    def l2_flush():
        flush.zero_()
        torch.cuda.synchronize()

    for _ in range(args.warmup):
        bf, log = B.factorize(op, rt, ct, rc)
    # ----------------------------------------------------------- timed
    barrier()
    clocks = ClockSampler(local)
    ctx.profile(-1)
    ctx.profile(1)
    launches0 = ctx.launches
    total_ms, flops, logs, step_ms = 0.0, 0.0, [], []
    for _ in range(args.steps):
        l2_flush()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        bf, log = B.factorize(op, rt, ct, rc)
        e1.record(stream)
        e1.synchronize()
        step_ms.append(e0.elapsed_time(e1))
        total_ms += step_ms[-1]
        flops += log.flops
        logs.append(log)
    launches = ctx.launches - launches0
    kernels = ctx.profile_report()
    ctx.profile(0)
    barrier()
    clk = clocks.stop()
    max_ms = allreduce(total_ms, "max")
    fl_total = allreduce(flops, "sum")
    value = fl_total / (max_ms / 1e3) / 1e9
    ms_per_step = max_ms / args.steps

    # ----------------------------------------------- apply bandwidth (device)
    def time_apply(bfx, ks, reps=10):
        """device-resident apply, L2 flushed before every call, CUDA events on the library stream"""
        out = {}
        nin, nout = bfx.cols, bfx.rows
        for k in ks:
            x = torch.randn((k, nin), dtype=torch.complex128, device="cuda").t()
            y = torch.empty((k, nout), dtype=torch.complex128, device="cuda").t()

            def call():
                B.api.check(B.api.lib().bfly_apply(bfx.h, 0, B.api.C.c_void_p(x.data_ptr()), nin,
                                                   B.api.C.c_void_p(y.data_ptr()), nout, k, 1))

            for _ in range(3):
                call()
            ts = []
            for _ in range(reps):
                l2_flush()
                a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a0.record(stream)
                call()
                a1.record(stream)
                a1.synchronize()
                ts.append(a0.elapsed_time(a1))
            ms = statistics.median(ts)
            nbytes = 16.0 * (bfx.nnz() + (nin + nout) * k)
            gbs = nbytes / (ms / 1e3) / 1e9
            out[f"k{k}"] = {"ms": round(ms, 4), "GB/s": round(gbs, 1), "frac_of_hbm": round(gbs / HBM_PEAK_GBS, 3),
                            "bytes": nbytes, "tflops": round(8.0 * bfx.nnz() * k / (ms / 1e3) / 1e12, 2)}
            del x, y
        return out

    # config 2's factorization (168 MB of factors) and config 4's input
    # butterfly (n = 262144, leaf 64, rank 32: 1.95 GB -- the HBM-bound case of SURVEY 8d)
    apply, apply4 = {}, {}
    if rank == 0:
        apply = time_apply(bf, (1, 2, 16))
        if not args.no_extra:
            bf4 = B.synth_butterfly(12, 32, 0, leaf=64, perturb=1e-8, ctx=ctx)
            apply4 = time_apply(bf4, (1, 16))
            apply4["nnz"] = bf4.nnz()
            del bf4

    # --------------------------------------------------- e2e (host buffers)
    import ctypes as C

    pts_t = torch.from_numpy(np.ascontiguousarray(op.targets)).pin_memory()
    pts_s = torch.from_numpy(np.ascontiguousarray(op.sources)).pin_memory()
    kappa = op.wavenumber
    e2e_steps = max(1, min(args.steps, 3))
    h2d = (pts_t.numel() + pts_s.numel()) * 8
    d2h = 0
    # the result lands in a reused pinned host buffer, as a serving pipeline would
    host_out = torch.empty(bf.serialized_size() + (1 << 20), dtype=torch.uint8, pin_memory=True)
    barrier()
    te0 = time.perf_counter()
    e2e_split = []
    for _ in range(e2e_steps):
        t0 = time.perf_counter()
        h = C.c_void_p()
        B.api.check(B.api.lib().bfly_op_kernel(ctx.h, B.api.OP_CIRCLE, op.rows, op.cols,
                                               C.c_void_p(pts_t.data_ptr()), C.c_void_p(pts_s.data_ptr()), kappa,
                                               B.api.COMPLEX128, C.byref(h)))
        op_e = B.api.BlackBoxOperator(h, ctx, B.api.COMPLEX128)
        bf_e, log_e = B.factorize(op_e, rt, ct, rc)
        t1 = time.perf_counter()
        if rank == 0 or not sharded:
            blob = bf_e.serialize(out=host_out.numpy())  # every factor block back on the host
            d2h = len(blob)
        t2 = time.perf_counter()
        e2e_split.append((round(t1 - t0, 4), round(t2 - t1, 4)))
        del bf_e, op_e  # the result now lives on the host; free its device copy before the next job
    barrier()
    te = (time.perf_counter() - te0) / e2e_steps
    e2e_val = (fl_total / args.steps) / te / 1e9  # whole-job flops of one construction

    # ------------------------------------------------------------ roofline
    # K2 (kernel_matvec): kernel entries evaluated on the FP64 pipe, complex128
    # contraction exact in int8 slices on tcgen05 (k_matvec_oz.cu).  `achieved`
    # = the algorithmic complex128 contraction flops (8 per complex MAC) per
    # launch / the launch's event time, against the native FP64 peak: the int8
    # emulation is what lets it exceed 1.  The int8 tensor ops the launch
    # actually executes are reported next to it against the measured int8 peak.
    mv = kernels.get("kernel_matvec", {"launches": 1, "ms": 1, "flops": 0, "bytes": 0})
    i8 = kernels.pop("kernel_matvec.int8_ops", None)
    achieved = mv["flops"] / (mv["ms"] / 1e3) / 1e12 if mv["ms"] > 0 else 0.0
    roofline = {
        "bound": "tensor",
        "kernel": "kernel_matvec (K2: kernel-entry evaluation on the FP64 pipe + exact int8-slice complex128 "
                  "contraction on tcgen05; FP64 and tensor ops time-share one datapath on B200)",
        "achieved": round(achieved, 3), "peak": FP64_PEAK_TFLOPS, "unit": "TFLOP/s",
        "frac": round(achieved / FP64_PEAK_TFLOPS, 4), "traffic": K2_DRAM_BYTES_PER_LAUNCH,
        "peak_source": "measured FP64 DMMA peak (tools/microbench/fp64_peaks.cu, profiles/r01_fp64_peaks.txt; "
                       "MEASURED_PEAKS.json has no FP64 entry); achieved = algorithmic complex128 contraction "
                       "flops, computed exactly via int8 slices, so frac > 1 is possible",
        "traffic_source": "ncu --set full, one config-2 transfer-level launch (profiles/r02_k2_ncu_s2.txt)",
        "flops_per_launch": mv["flops"] / max(1, mv["launches"]), "avg_launch_ms": mv["ms"] / max(1, mv["launches"]),
        "share_of_step": round(mv["ms"] / total_ms, 4) if total_ms else None,
    }
    if i8 and i8["ms"] > 0:
        tops = i8["flops"] / (i8["ms"] / 1e3) / 1e12
        roofline["int8"] = {"achieved_tops": round(tops, 1), "peak_tops": INT8_PEAK_TOPS,
                            "frac": round(tops / INT8_PEAK_TOPS, 4),
                            "peak_source": "measured tcgen05 kind::i8 M128 N256 (tools/microbench/tc_i8.cu)"}
    roofline["pipes_busy"] = dict(K2_PIPES, source="ncu --set full sm__pipe_*_cycles_active, one config-2 "
                                                   "transfer-level launch (profiles/r02_k2_ncu_s2.txt); FP64 "
                                                   "and int8 tensor ops time-share one datapath "
                                                   "(profiles/r01_tc_i8.txt overlap test)")

    # ------------------------------- the other full-size configs (info only)
    # config 4 (recompression, n = 262144: the north-star scaling config) and
    # config 1 (3D plates, n = 16384): one warm-up + median of 3 constructions
    # (own context: its memory pool does not disturb the timed legs above)
    other = {}
    if rank == 0 and world == 1 and not args.no_extra:
        ctx_x = B.Context(local)
        for cid in (4, 1):
            wx = B.configs.build(cid, ctx=ctx_x)
            ts_x = []
            for i in range(4):
                l2_flush()
                bx, lx = B.factorize(wx.op, wx.row_tree, wx.col_tree, wx.recon)
                if i:
                    ts_x.append(lx.total_seconds)
            med = statistics.median(ts_x)
            # flops = the ones executed (config 4's butterfly black box skips the blocks a
            # structured probe's zero rows cannot reach and answers the basis projection itself: 1.0 TFLOP instead of the padded 18.7)
            other[wx.name] = {"construct_s": round(med, 4), "GFLOP/s": round(lx.flops / med / 1e9, 1),
                              "TFLOP_executed": round(lx.flops / 1e12, 3), "max_rank": bx.max_rank(), "nnz": bx.nnz()}
            if cid == 4:
                # the same factorization through the reference's padded products (BFLY_NO_STRUCT_APPLY=1)
                # executes 18.67 TFLOP in 0.715 s on this GPU (profiles/r02_cfg4_structured.txt)
                other[wx.name]["padded_reference_path"] = {"TFLOP": 18.67, "construct_s": 0.715}
            del bx, wx
        del ctx_x

    if rank == 0:
        line = {
            "metric": METRIC, "value": round(value, 3), "unit": "GFLOP/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(ms_per_step, 3), "higher_is_better": True,
            "scaling": "strong" if sharded else "weak", "vs_baseline": None, "dtype": "complex128",
            "data": "synthetic",
            "config": {"workload": "config2_helmholtz_circle_n65536", "n": w.n, "levels": rc.levels, "leaf": 32,
                       "tol": rc.tolerance, "r0": rc.rank_guess, "oversampling": rc.oversampling,
                       "parallelism": (f"probe-sharded x{world} ({transport} all-gather per level)" if sharded
                                       else f"replicas{world}" if world > 1 else "single"),
                       "transport": transport if world > 1 else None,
                       "l2": "flushed before every step (256 MB write); probe products 0.1-1 GB > L2"},
            "construct_seconds": round(ms_per_step / 1e3, 4),
            "construct_seconds_median": round(statistics.median(step_ms) / 1e3, 4),
            # per-phase wall times (PhaseStat names), median over the timed steps
            "phases_ms": {p.name: round(statistics.median(lg.phases[i].seconds for lg in logs) * 1e3, 3)
                          for i, p in enumerate(logs[0].phases)},
            "flops_per_step": fl_total / args.steps, "kernel_evals_per_step": logs[0].kernel_evals,
            "max_rank": bf.max_rank(), "nnz": bf.nnz(),
            "k2_fp64_recomputes": sum(int(lg.products_recomputed) for lg in logs),
            "roofline": roofline,
            "apply": apply,
            "apply_cfg4": apply4,
            "other_configs": other,
            "kernels": {k: {"launches": v["launches"], "ms_per_step": round(v["ms"] / args.steps, 3)}
                        for k, v in kernels.items()},
            "e2e": {"value": round(e2e_val, 3), "unit": "GFLOP/s", "h2d_bytes_per_step": int(h2d),
                    "d2h_bytes_per_step": int(d2h), "seconds_per_step": round(te, 4),
                    "steps_s": e2e_split},
            "gpu_launches": int(launches),
            "clocks": clk,
        }
        if world == 1 and not args.no_cpu:
            # a bounded sample of ~10-30 s of CPU work (two reference-arm steps)
            v, dt, threads, kind, sample = cpu_sample(probes=2 * args.ref_probes)
            line["cpu_baseline"] = {"value": round(v, 3), "unit": "GFLOP/s", "cores": threads, "kind": kind,
                                    "sample": sample, "seconds": round(dt, 2), "scope": SAMPLE_SCOPE,
                                    "full_construction": full_reference_construction()}
        print(json.dumps(line), flush=True)
    if dist is not None:
        dist.barrier()
        dist.destroy_process_group()
    return 0


def _free_port():
    import socket

    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def self_launch(args, argv):
    """--gpus N > 1 without a torchrun environment: launch N ranks (one
    process per GPU) under torch.distributed.run on this node."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()), os.path.abspath(__file__)] + argv
    print(f"bench: launching {args.gpus} ranks: {' '.join(cmd[1:])}", file=sys.stderr, flush=True)
    return subprocess.call(cmd)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--size", type=int, default=0, help="override n (testing only)")
    ap.add_argument("--ref-probes", type=int, default=8)
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-extra", action="store_true", help="skip the other full-size configs (info only)")
    ap.add_argument("--mode", default="shard", choices=["shard", "replica"], help="N > 1 schedule")
    ap.add_argument("--transport", default="auto", choices=["auto", "nccl", "host"],
                    help="N > 1 exchange: NCCL (one GPU per rank) or host-staged over gloo (ranks may share "
                         "a GPU: a correctness run, not a scaling measurement); auto = NCCL when every rank "
                         "has its own GPU")
    ap.add_argument("--dry-launch", action="store_true", help="print rank/world and exit (launcher test)")
    argv = sys.argv[1:]
    args = ap.parse_args(argv)
    if args.gpus < 1:
        ap.error("--gpus must be >= 1")
    env_world = os.environ.get("WORLD_SIZE")
    if env_world is None and args.gpus > 1:
        return self_launch(args, argv)
    if env_world is not None and int(env_world) != args.gpus:
        print(f"bench: refusing to run: --gpus {args.gpus} but WORLD_SIZE={env_world}", file=sys.stderr, flush=True)
        return 2
    if args.dry_launch:
        rank, world, local = _env_rank()
        print(json.dumps({"rank": rank, "world": world, "local_rank": local}), flush=True)
        return 0
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
