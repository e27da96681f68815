"""K2 alone on a fixed workload: the config-2 operator (n = 65536, Helmholtz
circle, complex128) applied to a device-resident 65536 x 32 probe block
(one dense product = 1.1 TFLOP of complex contraction), N / H; prints the
K2 device time per launch from the library's CUDA-event profile.  Used for
same-box A/B of library builds (BFLY_LIB) and experiment builds whose
results are not meaningful (the workload does not depend on them)."""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2002_03400_b200 as B  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--cfg", type=int, default=2)
    ap.add_argument("--cols", type=int, default=32)
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--modes", default="NH", help="N and/or H")
    a = ap.parse_args()
    w = B.configs.build(a.cfg)
    n = w.op.cols
    g = torch.Generator(device="cuda").manual_seed(0)
    x = torch.randn(a.cols, n, dtype=torch.complex128, device="cuda", generator=g).t()  # column-major
    for name in a.modes:
        f = w.op.apply if name == "N" else w.op.apply_adjoint
        f(x)
        torch.cuda.synchronize()
        w.op.ctx.profile(-1)
        w.op.ctx.profile(1)
        for _ in range(a.reps):
            f(x)
        torch.cuda.synchronize()
        rep = w.op.ctx.profile_report()
        k = rep.get("kernel_matvec", {})
        ms = k.get("ms", 0.0) / max(1, k.get("launches", 1))
        tf = k.get("flops", 0.0) / max(k.get("ms", 1e-9), 1e-9) / 1e9
        print(f"cfg {a.cfg} {name}: K2 {ms:.3f} ms per launch, {tf:.2f} TF/s (complex128-equivalent)")
        w.op.ctx.profile(0)


if __name__ == "__main__":
    main()
