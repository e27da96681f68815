// k_eval.cuh -- on-the-fly kernel-entry evaluation shared by the K2 matvec
// kernels (FP64 DMMA path k_matvec.cu and integer-slice tensor path
// k_matvec_oz.cu).  Entry formulas follow the oracle (oracle/bo_operators.c,
// the BASELINE operators of SURVEY App. A) with r, the phase and 1/r
// bit-identical to it; sin/cos differ by ulps.
#pragma once

#include "common.cuh"
#include "kernels.cuh"

namespace bfly {
namespace keval {

constexpr double kTwoPi = 6.283185307179586476925286766559;
constexpr double kFourPi = 12.566370614359172953850573533118;

// sin/cos of an argument reduced by the 2-term FMA Cody-Waite step (|ph| up to
// ~1e5 here) and evaluated with Taylor polynomials on [-pi/4, pi/4]
// (truncation < 1e-19); ~20 FP64 ops instead of ~47 for libdevice sincos.
// Taylor coefficients in the constant bank: DFMA reads c[][] operands
// directly (64-bit immediates would be re-materialised with UMOVs).
static __constant__ double kSinC[8] = {2.8114572543455207632e-15,  -7.6471637318198164759e-13,   // 1/17!, -1/15!
                                1.6059043836821614599e-10,  -2.5052108385441718775e-08,   // 1/13!, -1/11!
                                2.7557319223985890653e-06,  -1.9841269841269841270e-04,   // 1/9!,  -1/7!
                                8.3333333333333333333e-03,  -1.6666666666666666667e-01};  // 1/5!,  -1/3!
static __constant__ double kCosC[8] = {4.7794773323873852974e-14,  -1.1470745597729724714e-11,   // 1/16!, -1/14!
                                2.0876756987868098979e-09,  -2.7557319223985890653e-07,   // 1/12!, -1/10!
                                2.4801587301587301587e-05,  -1.3888888888888888889e-03,   // 1/8!,  -1/6!
                                4.1666666666666666667e-02,  -0.5};                        // 1/4!,  -1/2!

__device__ __forceinline__ void sincos_red(double f, int q, double& s, double& c) {
  const double x2 = f * f;
  double ps = kSinC[0], pc = kCosC[0];
#pragma unroll
  for (int i = 1; i < 8; ++i) {
    ps = fma(ps, x2, kSinC[i]);
    pc = fma(pc, x2, kCosC[i]);
  }
  const double sn = fma(f * x2, ps, f);
  const double cs = fma(x2, pc, 1.0);
  // quadrant q mod 4: (s, c) <- (s, c), (c, -s), (-s, -c), (-c, s)
  const bool swap = q & 1;
  double rs = swap ? cs : sn, rc = swap ? sn : cs;
  if ((q + 1) & 2) rc = -rc;
  if (q & 2) rs = -rs;
  s = rs;
  c = rc;
}

__device__ __forceinline__ void fast_sincos(double ph, double& s, double& c) {
  const double q = rint(ph * 0.63661977236758134308);    // 2/pi
  double f = fma(-q, 1.5707963267948965580, ph);         // pi/2 high
  f = fma(-q, 6.1232339957367658e-17, f);                // pi/2 low
  sincos_red(f, (int)(long long)q, s, c);
}

// 1/r to ~1 ulp: MUFU.RCP64H seed + two Newton steps (amplitude only; the
// phase uses the correctly rounded r).
__device__ __forceinline__ double fast_rcp(double r) {
  double y;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(r));
  double e = fma(-r, y, 1.0);
  y = fma(y, e, y);
  e = fma(-r, y, 1.0);
  return fma(y, e, y);
}

template <int KIND>
__device__ __forceinline__ double2 kernel_entry_fast(double tx, double ty, double tz, double sx, double sy, double sz,
                                                     double kappa) {
  double sn, cs;
  if (KIND == KK_NUFFT) {
    // exp(2 pi i x xi): t = x xi, f = t - rint(t) in [-1/2, 1/2]; quarter turns exact
    const double ph = __dmul_rn(tx, sx);
    const double f = __dsub_rn(ph, rint(ph));
    const double qq = rint(4.0 * f);
    const double g = __dsub_rn(f, 0.25 * qq);
    sincos_red(__dmul_rn(kTwoPi, g), (int)qq, sn, cs);
    return make_double2(cs, sn);
  } else if (KIND == KK_PLATES) {
    const double dx = __dsub_rn(tx, sx), dy = __dsub_rn(ty, sy), dz = __dsub_rn(tz, sz);
    const double r = __dsqrt_rn(fma(dz, dz, fma(dy, dy, __dmul_rn(dx, dx))));
    fast_sincos(__dmul_rn(kappa, r), sn, cs);
    const double sc = fast_rcp(__dmul_rn(kFourPi, r));
    return make_double2(cs * sc, sn * sc);
  } else {
    const double dx = __dsub_rn(tx, sx), dy = __dsub_rn(ty, sy);
    const double r = __dsqrt_rn(fma(dy, dy, __dmul_rn(dx, dx)));
    fast_sincos(__dmul_rn(kappa, r), sn, cs);
    const double sc = fast_rcp(r);
    return make_double2(cs * sc, sn * sc);
  }
}


// ---- table-based sin/cos (K2 integer-slice path): 2048 table points over a
// full turn (tab[j] = (cos, sin)(2 pi j / 2048), in shared memory) and short
// polynomials on |f| <= pi/2048.  sin f = f - f^3/6 (the f^5/120 term is
// < 7.3e-17, 100x below the 2^-47 rounding of the sliced entries), cos f - 1 =
// f^2 (-1/2 + f^2/24) (f^6/720 < 2e-20).  Round 1 used 512 points and one more
// polynomial term: the 2048-point table saves one DFMA per entry (the
// evaluation's FP64 work is on K2's critical path: a table-free polynomial
// sin/cos measured 333 vs 300 ms per construction).
// kTabC: 2048/(2 pi), (2 pi/2048) high / low, -, -1/6, -, 1/24
constexpr int kTabN = 2048;
static __constant__ double kTabC[8] = {325.94932345220167, 0.0030679615757712823, 1.195944139792337e-19,
                                       0.0, -1.6666666666666666667e-01, 0.0, 4.1666666666666666667e-02, 0.0};
constexpr double kMagic = 6755399441055744.0;  // 1.5 * 2^52

// (s, c) of the angle a_j + f given the table entry (cos a_j, sin a_j)
__device__ __forceinline__ void tab_poly(double f, double2 tc, double& s, double& c) {
  const double f2 = f * f;
  const double sf = fma(f * f2, kTabC[4], f);
  const double pc = fma(f2, kTabC[6], -0.5);
  const double cm1 = f2 * pc;
  s = fma(tc.x, sf, fma(tc.y, cm1, tc.y));
  c = fma(-tc.y, sf, fma(tc.x, cm1, tc.x));
}

// sin/cos of a phase |ph| < 2^40
__device__ __forceinline__ void tab_sincos(double ph, const double2* __restrict__ tab, double& s, double& c) {
  const double t = fma(ph, kTabC[0], kMagic);
  const int qi = __double2loint(t);
  const double q = t - kMagic;
  double f = fma(-q, kTabC[1], ph);
  f = fma(-q, kTabC[2], f);
  tab_poly(f, tab[qi & (kTabN - 1)], s, c);
}

// exp(2 pi i g) for a reduced turn fraction f in [-1/2, 1/2]
__device__ __forceinline__ void tab_sincos_turn(double f, const double2* __restrict__ tab, double& s, double& c) {
  const double t = fma(f, (double)kTabN, kMagic);
  const int qi = __double2loint(t);
  const double g = __dsub_rn(f, (t - kMagic) * (1.0 / kTabN));  // exact (Sterbenz)
  tab_poly(__dmul_rn(kTwoPi, g), tab[qi & (kTabN - 1)], s, c);
}

// r = sqrt_rn(x) (bit-identical to __dsqrt_rn: 0 mismatches in 8.6e9 random
// normal inputs, tools/microbench/sqrt_check.cu) and h = 1/(2 sqrt(x)) to
// ~3 ulp as a by-product; branch-free Goldschmidt iteration + Markstein
// correction, positive normal x only (0 / inf / NaN yield non-finite h).
__device__ __forceinline__ double sqrt_rcp(double x, double& h) {
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  double s = x * y;
  h = __hiloint2double(__double2hiint(y) - (1 << 20), __double2loint(y));  // 0.5 y: exponent - 1 (integer pipe)
  double e = fma(-s, h, 0.5);
  s = fma(s, e, s);
  h = fma(h, e, h);
  e = fma(-s, h, 0.5);
  s = fma(s, e, s);
  h = fma(h, e, h);
  const double d = fma(-s, s, x);
  return fma(d, h, s);
}
}  // namespace keval
}  // namespace bfly
