// k_matvec_oz.cu -- K2 on the 5th-generation tensor cores: kernel-evaluated
// black-box products (reference operators.hpp:430-439 pattern, probe_with
// reconstruct.hpp:72-85) with the complex128 contraction done EXACTLY in
// integer arithmetic on tcgen05 kind::i8 (an Ozaki-style slice scheme).
//
// Why: on B200 the FP64 DMMA and DFMA share one 37 TF/s pipe
// (profiles/r01_fp64_peaks.txt), so in the FP64 path (k_matvec.cu) the
// ~43-instruction kernel-entry evaluation competes with the contraction.
// Here the FP64 pipe only evaluates entries; the contraction runs on the
// int8 tensor cores (4.2 POPS measured, tools/microbench/tc_i8.cu).
//
// Arithmetic (per CTA: 128 output rows x 32 complex probe columns), with the
// default 6-slice scheme (BFLY_OZ_SLICES=7 restores the round-1 scheme):
//  * every kernel entry a (re and im separately) is scaled by 2^S_row and
//    rounded to a signed integer |v| < 2^47; S_row is per output row and per
//    2048-entry chunk of the input range, from a bound on |a| over the chunk
//    (1 for NUFFT, 1/r_min or 1/(4 pi r_min) for the Helmholtz kernels);
//  * v's two's-complement bytes ARE its base-256 digits: slices A_0..A_4
//    unsigned, A_5 signed -- no decomposition work;
//  * probe entries x are scaled per column by 2^T_c (|x| < 2^46) and split into
//    balanced signed digits B_0..B_5 (prep kernel, once per launch);
//  * sum_k v_ik w_kc = sum_{p,q} 2^{8(p+q)} A_p B_q^T; the products with
//    p + q >= 4 (26 of 36 slice pairs) are accumulated exactly in int32 in
//    TMEM, one 64-column block per diagonal e = p + q (7 blocks = 448 cols).
//    The dropped terms are < 2^-52 relative to max|v| max|w| per entry, the
//    rounding to integers 2^-47 / 2^-46 relative to the row / column bound.
//    (`BFLY_OZ_E0=5`, an experiment build, also drops e = 4: 21 pairs, 19 %
//    less tensor work, 7 % less K2 time, but < 2^-43.6 per entry -- the
//    black-box products of the Helmholtz circle then differ from the FP64
//    oracle by ~3e-12 at n = 1024 instead of ~1e-14: not kept.)
//  * every chunk the diagonals are drained into FP64 accumulators (Horner in
//    2^8, times 2^{8 E0 - S_row - T_c}).
// Complex: A_re slices multiply G1 = [B(Re x) | B(Im x)] and A_im slices
// multiply G2 = [B(-Im x) | B(Re x)] into the same accumulator, so TMEM block
// columns hold [Re y | Im y] directly.  For slice A_p the needed B_q
// (q = e - p) form a contiguous window of the concatenated B slices, so one
// MMA covers up to four diagonals.
//
// Pipeline (1 CTA / SM, TMEM fully allocated): 16 evaluation warps write A
// stages (128 rows x 32 input entries, both planes) into a double-buffered
// shared-memory ring and drain TMEM; one thread issues the B-stage bulk
// copies; one thread of warp 16 issues the MMAs and commits them to mbarriers.
//
// Safety: if any scaled entry falls outside the representable range (a
// coincident point, a bound that did not hold) the launch reports it and the
// caller recomputes the product with the FP64 DMMA kernel.
#include <algorithm>
#include <atomic>
#include <cstdio>
#include <cstdlib>
#include <string>
#include <vector>

#include "k_eval.cuh"
#include "kernels.cuh"

namespace bfly {

namespace {

// Slice scheme (BFLY_OZ_SLICES): 6 slices per operand, |v| < 2^47 (A, two's
// complement bytes) and |x| < 2^46 (B, balanced digits), diagonals e >= 4 kept
// (26 slice-pair products; dropped terms < 2^-53 relative); or 7 slices,
// |v|, |x| < 2^50, e >= 5 kept (34 products; dropped < 2^-50 relative).
#ifndef BFLY_OZ_SLICES
#define BFLY_OZ_SLICES 6
#endif
constexpr int OZ_NSL = BFLY_OZ_SLICES;            // slices per operand
static_assert(OZ_NSL == 6 || OZ_NSL == 7, "6 or 7 slices");
// lowest kept diagonal e = p + q: NSL - 2 (6 slices: e >= 4, 26 slice pairs,
// 7 diagonals) or NSL - 1 (BFLY_OZ_E0 = 5, experiment: 21 pairs, 6 diagonals)
#ifndef BFLY_OZ_E0
#define BFLY_OZ_E0 (BFLY_OZ_SLICES - 2)
#endif
constexpr int OZ_E0 = BFLY_OZ_E0;
static_assert(OZ_E0 == OZ_NSL - 1 || OZ_E0 == OZ_NSL - 2, "kept diagonals");
constexpr int OZ_NDIAG = 2 * OZ_NSL - 1 - OZ_E0;  // kept diagonals e = E0 .. 2 NSL - 2
constexpr int OZ_ABITS = OZ_NSL == 6 ? 47 : 50;   // |v| < 2^ABITS (scaled, rounded kernel entries)
constexpr int OZ_BBITS = OZ_NSL == 6 ? 46 : 50;   // |x| < 2^BBITS (scaled, rounded probe entries)
constexpr int OZ_KS = 32;                         // input entries per stage (MMA K)
// drain / scale chunk: 2048 entries (int32 diagonal sums stay < 2^30); the 3D
// kernel keeps 1024 (its z coordinates must fit shared memory too)
constexpr int oz_kd(int kind) { return kind == KK_PLATES ? 1024 : 2048; }
constexpr int OZ_NST = 2;                         // ring depth
constexpr int OZ_BM = 128;                        // output rows per CTA (= TMEM lanes)
constexpr int OZ_EWARPS = 16;                     // CTA-pair kernel: evaluation warps
constexpr int OZ_THREADS = OZ_EWARPS * 32;        // evaluation threads
constexpr int OZ_EPT = OZ_BM * OZ_KS / OZ_THREADS;  // 8 entries per thread per stage
// single-CTA kernel: OZS_WARPS evaluation warps, OZS_EPT entries per thread per stage
#ifndef OZ_EW
#define OZ_EW 16
#endif
#ifndef OZ_DEFER
#define OZ_DEFER 1  // the last warp to write a stage issues its MMAs after its share of the next one
#endif
#ifndef OZ_LB_PAD
#define OZ_LB_PAD 0  // experiment: launch-bounds padding (register cap) of the single-CTA kernel
#endif
constexpr int OZS_WARPS = OZ_EW;
constexpr int OZS_THREADS = OZS_WARPS * 32;
constexpr int OZS_EPT = OZ_BM * OZ_KS / OZS_THREADS;  // 8 or 16
static_assert(OZS_EPT == 8 || OZS_EPT == 16, "single-kernel thread mapping");
constexpr int OZ_ASLICE = OZ_BM * OZ_KS;           // 4096 B: one A slice (128 rows x 32 B)
constexpr int OZ_APLANE = OZ_NSL * OZ_ASLICE;      // 24576 B
constexpr int OZ_ASTAGE = 2 * OZ_APLANE;           // re + im planes
// A stage layout (both kernels, and the evaluation cache): [K-half][plane][slice]
// blocks of 128 rows x 16 B (2 KB; core matrices of 8 rows x 16 B, 128 B
// apart), so the MMA descriptor's K step (LBO) is half a stage and a stage
// is one contiguous 48 KB image
constexpr int OZ_AHALF = OZ_ASTAGE / 2;            // 24 KB: one K-half of a stage
constexpr int OZ_ABLK = OZ_AHALF / (2 * OZ_NSL);   // 2 KB: one (plane, slice) block of a K-half
constexpr int OZ_MAXCB = 64;                       // stride of the per-tile column scales
constexpr int OZ_MAXCB1 = 32;                      // widest probe tile of the single-CTA kernel
static_assert(OZ_EPT == 8, "thread mapping assumes 8 entries per thread");

constexpr int pow2_ceil(int x) { return x <= 32 ? 32 : x <= 64 ? 64 : x <= 128 ? 128 : x <= 256 ? 256 : 512; }

// Per-stage MMA schedule.  Plane h (0: A_re x G1, 1: A_im x G2), slice p,
// first diagonal block jlo, block count nb (N = BN2 nb <= 256), init (first
// K-step of a chunk writes instead of accumulating).  Diagonal block j holds
// e = p + q = j + E0, so slice A_p meets B_q for the blocks j with
// q = j + E0 - p in [0, NSL) -- a contiguous window of the concatenated B
// slices.
// OZ_ZERO_ACC (default): the warps that drain a chunk write zeros back into
// the TMEM they read (and zero it at kernel start), so every MMA accumulates
// and each slice's block range splits freely into windows of <= 256 columns
// (18 MMAs per stage instead of 20; tools/microbench/tc_tmem_a.cu: 1796 vs
// 1933 cycles per stage alone).  Otherwise the initialising MMAs (plane 0)
// come first and cover every block exactly once: the top slice misses block
// 0 (with E0 = NSL - 2), which the next slice's first MMA initialises.
//   packed: h | p << 1 | jlo << 4 | nb << 8 | init << 13
#ifndef OZ_ZERO_ACC
#define OZ_ZERO_ACC 1
#endif
#ifndef OZ_GACC
#define OZ_GACC 1
#endif
// timing experiments only (wrong results): bit 0 skips the MMAs, bit 1 the
// kernel-entry evaluation, bit 2 the B refills, bit 3 the A-slice writes
// (tools/k2_bench.py with an experiment build)
#ifndef OZ_EXP
#define OZ_EXP 0
#endif
// mbarrier waits with a suspend-time hint (round 2) or a plain try_wait
// loop (default: 18.8 vs 19.5 ms per dense config-2 product)
#ifndef OZ_WAIT_HINT
#define OZ_WAIT_HINT 0
#endif


struct OzSched {
  uint32_t code[64];
  int n;
};
constexpr uint32_t mma_code(int h, int p, int jlo, int nb, int init) {
  return (uint32_t)(h | (p << 1) | (jlo << 4) | (nb << 8) | (init << 13));
}
constexpr OzSched make_sched(int maxb) {
  OzSched sc{};
  sc.n = 0;
  constexpr int T = OZ_NSL - 1, D = OZ_NDIAG;
  for (int h = 0; h < 2; ++h) {
    const int init = h == 0 ? 1 : 0;
    if (OZ_ZERO_ACC || OZ_E0 == OZ_NSL - 1) {
      // slice p meets blocks max(0, p - E0) .. min(D - 1, T + p - E0); with
      // E0 = NSL - 1 the top slice meets every block and initialises them
      for (int p = T; p >= 0; --p) {
        const int jlo = p > OZ_E0 ? p - OZ_E0 : 0;
        const int jhi = (D - 1) < (T + p - OZ_E0) ? (D - 1) : (T + p - OZ_E0);
        for (int j = jlo; j <= jhi; j += maxb)
          sc.code[sc.n++] = mma_code(h, p, j, (jhi + 1 - j) < maxb ? jhi + 1 - j : maxb,
                                     (!OZ_ZERO_ACC && p == T) ? init : 0);
      }
    } else {
      for (int j = 1; j <= D - 1; j += maxb) sc.code[sc.n++] = mma_code(h, T, j, (D - j) < maxb ? D - j : maxb, init);
      sc.code[sc.n++] = mma_code(h, T - 1, 0, 1, init);
      for (int j = 1; j <= T; j += maxb) sc.code[sc.n++] = mma_code(h, T - 1, j, (T + 1 - j) < maxb ? T + 1 - j : maxb, 0);
      for (int p = T - 2; p >= 0; --p)
        for (int j = 0; j <= p + 1; j += maxb) sc.code[sc.n++] = mma_code(h, p, j, (p + 2 - j) < maxb ? p + 2 - j : maxb, 0);
    }
  }
  return sc;
}

// NCB-dependent sizes and the shared-memory map (bytes)
template <int NCB_, int KD_, bool HASZ_>
struct OzT {
  static constexpr int NCB = NCB_;                   // complex probe columns per tile
  static constexpr int KD = KD_;                     // entries per drain / scale chunk
  static constexpr int NBOX = KD / 32;               // sub-boxes of 32 points per chunk
  static constexpr int BN2 = 2 * NCB;                // N-rows per B slice ([re | im])
  static constexpr int TMEM_COLS = pow2_ceil(OZ_NDIAG * BN2);
  static constexpr int BROWS = OZ_NSL * BN2;         // N-rows per B operand
  static constexpr int BOPER = BROWS * OZ_KS;        // G1 or G2 image
  static constexpr int BSTAGE = 2 * BOPER;           // G1 + G2
  static constexpr int MAXB = 256 / BN2 < OZ_NDIAG ? 256 / BN2 : OZ_NDIAG;  // blocks per MMA
  static constexpr int DC = NCB / 2;                 // drained columns per thread
  static constexpr int SM_A = 0;
  static constexpr int SM_B = SM_A + OZ_NST * OZ_ASTAGE;
  static constexpr int SM_PD = SM_B + OZ_NST * BSTAGE;  // double2 (x, y) [KD]
  static constexpr int SM_PZ = SM_PD + KD * 16;         // double z [KD] (3D kernels only)
  static constexpr int SM_S = SM_PZ + (HASZ_ ? KD * 8 : 0);  // int S_row [2][128]
  static constexpr int SM_T = SM_S + 2 * OZ_BM * 4;     // int T [NCB]
  static constexpr int SM_MIN = SM_T + OZ_MAXCB * 4;    // uint min d2 bits [128]
  static constexpr int SM_TAB = SM_MIN + OZ_BM * 4;     // double2 sin/cos table [kTabN]
  static constexpr int SM_BOX = SM_TAB + keval::kTabN * 16;  // float4 sub-box bounds [NBOX][2]
  static constexpr int SM_CNT = SM_BOX + NBOX * 32;     // uint stage arrival counters [NST]
  static constexpr int SM_BAR = SM_CNT + 16;            // mbarriers
  static constexpr int NBAR = 3 * OZ_NST + 1;  // fullB, empty, acc_full (+ fullA: the pair kernel)
  static constexpr int SM_TMEM = SM_BAR + NBAR * 8;
  static constexpr int SM_TOTAL = SM_TMEM + 16;
  static_assert(SM_TOTAL <= 232448, "shared memory budget");
  static_assert(NCB % 8 == 0 && NCB <= OZ_MAXCB, "tile width");
};

struct OzItem {
  int64_t row0, rows;   // input point range
  int64_t x_off, ldx;   // probe block
  int64_t ycol, ybase;  // output column, split-K slice base
  int64_t bstage0;      // first B stage image of this item
  int32_t ncols, pad_;
};

// ------------------------------------------------------------ PTX helpers
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ uint64_t smem_desc(uint32_t addr, uint32_t lbo, uint32_t sbo) {
  // K-major, SWIZZLE_NONE canonical layout; version 1 (sm_100)
  return (uint64_t)((addr >> 4) & 0x3FFF) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | ((uint64_t)1 << 46);
}
__host__ __device__ constexpr uint32_t idesc_i8(int M, int N, bool a_signed, bool b_signed) {
  return (2u << 4) | ((a_signed ? 1u : 0u) << 7) | ((b_signed ? 1u : 0u) << 10) | ((uint32_t)(N >> 3) << 17) |
         ((uint32_t)(M >> 4) << 24);
}
__device__ __forceinline__ void mma_i8(uint32_t d, uint64_t da, uint64_t db, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(d),
      "l"(da), "l"(db), "r"(idesc), "r"(acc));
}
// one lane of a converged warp (elect.sync)
__device__ __forceinline__ bool elect_one() {
  uint32_t pred = 0;
  asm volatile(
      "{\n\t.reg .pred P;\n\telect.sync _|P, 0xffffffff;\n\tselp.b32 %0, 1, 0, P;\n\t}\n"
      : "=r"(pred));
  return pred != 0;
}
// a value the compiler may keep in a uniform register (lane 0's, broadcast)
__device__ __forceinline__ uint32_t warp_uniform(uint32_t v) { return __shfl_sync(0xffffffffu, v, 0); }
__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.release.cta.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
#if OZ_WAIT_HINT
  // suspend-time hint: a waiting warp sleeps until the phase completes
  // instead of spinning on issue slots the MMA-issuing warp needs
  asm volatile(
      "{\n\t.reg .pred done;\n\t"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.acquire.cta.shared::cta.b64 done, [%0], %1, %2;\n\t"
      "@!done bra WAIT_%=;\n\t}\n" ::"r"(bar),
      "r"(parity), "r"(1000000u)
      : "memory");
#else
  asm volatile(
      "{\n\t.reg .pred done;\n\t"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.acquire.cta.shared::cta.b64 done, [%0], %1;\n\t"
      "@!done bra WAIT_%=;\n\t}\n" ::"r"(bar),
      "r"(parity)
      : "memory");
#endif
}
__device__ __forceinline__ void mma_commit(uint32_t bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
               "l"(src), "r"(bytes), "r"(bar)
               : "memory");
}
#ifdef OZ_TRACE
__device__ unsigned long long g_oz_trace[8];
// trace-build experiment switches (BFLY_OZ_MODE): 1 skip the MMAs, 2 skip the entry evaluation
__device__ int g_oz_mode;
#define OZT_BEGIN(v) const long long v = clock64();
#define OZT_END(v, slot) atomicAdd(&g_oz_trace[slot], (unsigned long long)(clock64() - v));
#else
#define OZT_BEGIN(v)
#define OZT_END(v, slot)
#endif

__device__ __forceinline__ void tmem_ld16(uint32_t addr, uint32_t (&v)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]), "=r"(v[8]),
        "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
      : "r"(addr));
}
__device__ __forceinline__ void tmem_ld4(uint32_t addr, uint32_t (&v)[4]) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0,%1,%2,%3}, [%4];"
               : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3])
               : "r"(addr));
}
// zeros into DC consecutive TMEM columns of the warp's lane quarter
template <int DC>
__device__ __forceinline__ void tmem_zero(uint32_t addr) {
  const uint32_t z = 0;
  if constexpr (DC % 16 == 0) {
#pragma unroll
    for (int q = 0; q < DC / 16; ++q)
      asm volatile(
          "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1};" ::"r"(
              addr + 16 * q),
          "r"(z)
          : "memory");
  } else {
#pragma unroll
    for (int q = 0; q < DC / 4; ++q)
      asm volatile("tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {%1,%1,%1,%1};" ::"r"(addr + 4 * q), "r"(z) : "memory");
  }
}
// exact int32 -> double (magic-number bias: one LOP + one DADD)
__device__ __forceinline__ double i2d(uint32_t v) {
  return __hiloint2double(0x43300000, (int)(v ^ 0x80000000u)) - 4503601774854144.0;  // 2^52 + 2^31
}
// x (|x| < 2^51) rounded to the nearest integer, as int64 (magic-number)
__device__ __forceinline__ long long d2ll(double x) {
  return __double_as_longlong(x + 6755399441055744.0) - 0x4338000000000000LL;  // 1.5 * 2^52
}
__device__ __forceinline__ double pow2(int e) { return __longlong_as_double((long long)(1023 + e) << 52); }

// 4x4 byte transpose: o[b] = byte b of w0..w3 (in order)
__device__ __forceinline__ void transpose4(uint32_t w0, uint32_t w1, uint32_t w2, uint32_t w3, uint32_t (&o)[4]) {
  const uint32_t t0 = __byte_perm(w0, w1, 0x5140), t1 = __byte_perm(w2, w3, 0x5140);
  const uint32_t t2 = __byte_perm(w0, w1, 0x7362), t3 = __byte_perm(w2, w3, 0x7362);
  o[0] = __byte_perm(t0, t1, 0x5410);
  o[1] = __byte_perm(t0, t1, 0x7632);
  o[2] = __byte_perm(t2, t3, 0x5410);
  o[3] = __byte_perm(t2, t3, 0x7632);
}

// kernel entry scaled by the row scale and rounded to an integer in one FMA
// each (magic-number rounding: result = value + 1.5 * 2^52); amp = scaled
// |entry| bound for the range check.  im is negated for the adjoint.
// NUFFT: the scale is p2 = 2^S.  Helmholtz kernels: the amplitude 1/r = 2h
// (1/(4 pi r) for the plates, whose table entries carry the 1/(4 pi)) times
// 2^S is h with S + 1 added to its exponent -- an integer add on the high
// word (es = (S + 1) << 20) instead of an FP64 multiply.
template <int KIND, bool CONJ>
__device__ __forceinline__ void entry_rounded(double tx, double ty, double tz, double sx, double sy, double sz,
                                              double kappa, double p2, int es, const double2* __restrict__ tab,
                                              double& re, double& im, double& amp) {
  double sn, cs, sc;
  if (KIND == KK_NUFFT) {
    const double ph = __dmul_rn(tx, sx);
    keval::tab_sincos_turn(__dsub_rn(ph, rint(ph)), tab, sn, cs);
    sc = p2;
  } else {
    const double dx = __dsub_rn(tx, sx), dy = __dsub_rn(ty, sy);
    double d2;
    if (KIND == KK_PLATES) {
      const double dz = __dsub_rn(tz, sz);
      d2 = fma(dz, dz, fma(dy, dy, __dmul_rn(dx, dx)));
    } else {
      d2 = fma(dy, dy, __dmul_rn(dx, dx));
    }
    double h;
    const double r = keval::sqrt_rcp(d2, h);
    keval::tab_sincos(__dmul_rn(kappa, r), tab, sn, cs);
    sc = __hiloint2double(__double2hiint(h) + es, __double2loint(h));
  }
  amp = sc;
  re = fma(cs, sc, keval::kMagic);
  im = fma(sn, CONJ ? -sc : sc, keval::kMagic);
}

// |v| < 2^ABITS <=> high word of the scaled amplitude below this (NaN / inf
// fail too).  The plates' amplitude sc = 2h 2^S omits the 1/(4 pi) that their
// table entries carry, so their limit is the high word of 4 pi 2^ABITS
// (truncated: a conservative bound)
template <int KIND>
__device__ __forceinline__ uint32_t amp_limit_hi() {
  return KIND == KK_PLATES ? (uint32_t)__double2hiint(keval::kFourPi * (double)(1ll << OZ_ABITS))
                           : (uint32_t)(1023 + OZ_ABITS) << 20;
}

// ------------------------------------------------------- probe slicing
// T_c = (BBITS - 1) - floor(log2 max_k |x_kc|_inf)  (scaled |x| < 2^BBITS)
__global__ void oz_colscale_kernel(const double2* __restrict__ X, const OzItem* __restrict__ items,
                                   int32_t* __restrict__ T) {
  const OzItem it = items[blockIdx.y];
  const int c = blockIdx.x;
  double m = 0.0;
  if (c < it.ncols)
    for (int64_t k = threadIdx.x; k < it.rows; k += blockDim.x) {
      const double2 v = X[it.x_off + k + (int64_t)c * it.ldx];
      m = fmax(m, fmax(fabs(v.x), fabs(v.y)));
    }
  __shared__ double red[256];
  red[threadIdx.x] = m;
  __syncthreads();
  for (int s = 128; s > 0; s >>= 1) {
    if (threadIdx.x < s) red[threadIdx.x] = fmax(red[threadIdx.x], red[threadIdx.x + s]);
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    const double mx = red[0];
    // zero or non-finite columns: scale 0 (non-finite values trip the slice check)
    T[blockIdx.y * OZ_MAXCB + c] = (mx > 0.0 && mx < 1e300) ? (OZ_BBITS - 1) - ilogb(mx) : 0;
  }
}

// balanced base-256 digits of round(x), |x| < 2^BBITS (the last one fits int8)
__device__ __forceinline__ void digits7(double x, int (&d)[OZ_NSL]) {
  long long q = d2ll(x);
#pragma unroll
  for (int s = 0; s < OZ_NSL - 1; ++s) {
    d[s] = (int)(signed char)(q & 0xFF);
    q = (q - d[s]) >> 8;
  }
  d[OZ_NSL - 1] = (int)q;
}

// one thread per (column c, 16-entry half of a stage): the balanced digits of
// round(x * 2^T_c) for those 16 input rows, written as whole 16-byte rows of
// the canonical K-major images of the stage (one N-row x 16 K per store):
//   G1 N-row q*BN2 + c:      Re x      G1 N-row q*BN2 + NCB + c:  Im x
//   G2 N-row q*BN2 + c:     -Im x      G2 N-row q*BN2 + NCB + c:  Re x
// (round 2 stored single bytes: 121 us per config-2 transfer level)
template <int NCB>
__global__ void oz_slice_kernel(const double2* __restrict__ X, const OzItem* __restrict__ items,
                                const int32_t* __restrict__ T, uint8_t* __restrict__ img, int* __restrict__ flag) {
  using Z = OzT<NCB, 1024, false>;  // B image geometry only (independent of KD)
  const OzItem it = items[blockIdx.y];
  const int64_t nst = ceil_div(it.rows, (int64_t)OZ_KS);
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= nst * 2 * NCB) return;
  const int c = (int)(t % NCB);
  const int kh = (int)((t / NCB) & 1);
  const int64_t st = t / (2 * NCB);
  const double sc = pow2(T[blockIdx.y * OZ_MAXCB + c]);
  constexpr double lim = (double)(1ll << OZ_BBITS);
  // digit s of entry j (j = 0..15) collected as bytes of 4 words per slice and part
  uint32_t wr[OZ_NSL][4], wi[OZ_NSL][4], wn[OZ_NSL][4];
#pragma unroll
  for (int q = 0; q < OZ_NSL; ++q)
#pragma unroll
    for (int w = 0; w < 4; ++w) wr[q][w] = wi[q][w] = wn[q][w] = 0;
  bool ok = true;
#pragma unroll
  for (int j = 0; j < 16; ++j) {
    const int64_t k = st * OZ_KS + kh * 16 + j;
    double2 v = make_double2(0.0, 0.0);
    if (c < it.ncols && k < it.rows) v = X[it.x_off + k + (int64_t)c * it.ldx];
    const double xr = v.x * sc, xi = v.y * sc;
    ok = ok && fabs(xr) < lim && fabs(xi) < lim;  // NaN fails too
    int dr[OZ_NSL], di[OZ_NSL], dn[OZ_NSL];
    digits7(xr, dr);
    digits7(xi, di);
    digits7(-xi, dn);
#pragma unroll
    for (int q = 0; q < OZ_NSL; ++q) {
      wr[q][j >> 2] |= (uint32_t)(dr[q] & 0xFF) << (8 * (j & 3));
      wi[q][j >> 2] |= (uint32_t)(di[q] & 0xFF) << (8 * (j & 3));
      wn[q][j >> 2] |= (uint32_t)(dn[q] & 0xFF) << (8 * (j & 3));
    }
  }
  if (!ok) {
    atomicOr(flag, 1);
    return;
  }
  uint8_t* g1 = img + (it.bstage0 + st) * (int64_t)Z::BSTAGE;
  uint8_t* g2 = g1 + Z::BOPER;
  auto row = [&](uint8_t* base, int nrow) {
    return reinterpret_cast<uint4*>(base + (kh * (Z::BROWS / 8) + (nrow >> 3)) * 128 + (nrow & 7) * 16);
  };
#pragma unroll
  for (int q = 0; q < OZ_NSL; ++q) {
    *row(g1, q * Z::BN2 + c) = make_uint4(wr[q][0], wr[q][1], wr[q][2], wr[q][3]);
    *row(g1, q * Z::BN2 + NCB + c) = make_uint4(wi[q][0], wi[q][1], wi[q][2], wi[q][3]);
    *row(g2, q * Z::BN2 + c) = make_uint4(wn[q][0], wn[q][1], wn[q][2], wn[q][3]);
    *row(g2, q * Z::BN2 + NCB + c) = make_uint4(wr[q][0], wr[q][1], wr[q][2], wr[q][3]);
  }
}

// sin/cos table (cos, sin)(2 pi j / kTabN), computed once per device: the
// per-CTA sincospi evaluation cost about one stage of FP64 work per CTA
// (1.5 % of the one-chunk CTAs of the deepest transfer levels)
__device__ double2 g_oz_tab[keval::kTabN];
__global__ void oz_table_kernel() {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j < keval::kTabN) {
    double s_, c_;
    sincospi(j / (keval::kTabN / 2.0), &s_, &c_);
    g_oz_tab[j] = make_double2(c_, s_);
  }
}

// ------------------------------------------------------------ main kernel
// Issue scheme: no dedicated MMA warp.  Each warp, after writing its part of
// an A stage, bumps the stage's arrival counter; the LAST warp to arrive
// issues the stage's MMAs (after the B bulk copy landed) and commits them to
// the slot's `empty` barrier (and, on a chunk's last stage, to `acc_full`).
// Chunk d-1 is drained by every warp BEFORE it arrives for stage 0 of chunk
// d, so the issuer of that stage knows TMEM is free.  tcgen05 MMAs of a CTA
// execute in issue order, so acc_full (committed by the last stage's
// issuer) covers the whole chunk.
template <int KIND, int MODE, int NCB>
__global__ void __launch_bounds__(OZS_THREADS + OZ_LB_PAD, 1)
    matvec_oz_kernel(Points outp, Points inp, double kappa, int64_t m_out, const uint8_t* __restrict__ bimg,
                     const int32_t* __restrict__ Tg, double2* __restrict__ Y, int64_t ldy,
                     const OzItem* __restrict__ items, int64_t rows_per_split, int64_t pstride, int* __restrict__ flag) {
  using Z = OzT<NCB, oz_kd(KIND), KIND == KK_PLATES>;
  extern __shared__ __align__(1024) uint8_t smem[];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  OZT_BEGIN(t5)
  const OzItem it = items[blockIdx.y];
  const int64_t i0 = (int64_t)blockIdx.x * OZ_BM;
  const int64_t kb = (int64_t)blockIdx.z * rows_per_split;
  const int64_t ke = min(it.rows, kb + rows_per_split);
  const int64_t nk = ke > kb ? ke - kb : 0;
  const int nchunks = (int)ceil_div(nk, (int64_t)Z::KD);

  double2* PD = reinterpret_cast<double2*>(smem + Z::SM_PD);
  double* PZ = reinterpret_cast<double*>(smem + Z::SM_PZ);
  int* Srow = reinterpret_cast<int*>(smem + Z::SM_S);
  int* Ts = reinterpret_cast<int*>(smem + Z::SM_T);
  unsigned* Smin = reinterpret_cast<unsigned*>(smem + Z::SM_MIN);
  unsigned* cnt = reinterpret_cast<unsigned*>(smem + Z::SM_CNT);
  const uint32_t bar0 = smem_u32(smem + Z::SM_BAR);
  auto fullB = [&](int s) { return bar0 + 8u * s; };
  auto empty = [&](int s) { return bar0 + 8u * (OZ_NST + s); };
  const uint32_t acc_full = bar0 + 8u * (2 * OZ_NST);
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + Z::SM_TMEM);

  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "n"(Z::TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 32) {
    for (int s = 0; s < OZ_NST; ++s) {
      mbar_init(fullB(s), 1);
      mbar_init(empty(s), 1);
      cnt[s] = 0;
    }
    mbar_init(acc_full, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (tid < NCB) Ts[tid] = Tg[blockIdx.y * OZ_MAXCB + tid];
  double2* tab = reinterpret_cast<double2*>(smem + Z::SM_TAB);
  for (int j = tid; j < keval::kTabN; j += OZS_THREADS) {  // L2-resident copy (plates: times 1/(4 pi))
    const double2 t = g_oz_tab[j];
    tab[j] = KIND == KK_PLATES ? make_double2(t.x * (1.0 / keval::kFourPi), t.y * (1.0 / keval::kFourPi)) : t;
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = *tmem_slot;
  const uint32_t sA = smem_u32(smem + Z::SM_A), sB = smem_u32(smem + Z::SM_B);

  // evaluation: row (warp & 7) * 16 + lane / 2, entries kofs .. kofs + EPT - 1 of each stage
  const int erow = (warp & 7) * 16 + (lane >> 1);
  const int kofs = OZS_EPT == 8 ? (warp >> 3) * 16 + (lane & 1) * 8 : (lane & 1) * 16;
  const int64_t gi = min(i0 + erow, m_out - 1);  // padded rows evaluate a valid row (never stored)
  const double ox = outp.x[gi];
  const double oy = KIND == KK_NUFFT ? 0.0 : outp.y[gi];
  const double oz = KIND == KK_PLATES ? outp.z[gi] : 0.0;
  // drain: TMEM lane quarter = warp & 3, column part dq = warp >> 2 of DC columns
  // (16 warps: Re y 0-15 / 16-31, Im y 0-15 / 16-31; 8 warps: Re y, Im y)
  const int drow = (warp & 3) * 32 + lane;
  const int dq = warp >> 2;
  constexpr int DC = OZS_WARPS == 16 ? Z::DC : NCB;
  constexpr int DPC = NCB / DC;  // column parts per component
  // the thread's output entries: row drow, columns (dq & 1) * DC + c of Re
  // (dq < 2) or Im y.  OZ_GACC (default): each chunk's drained sums are added
  // straight into them (a read-modify-write once per 64 stages; every entry
  // has one owner), which frees the DC FP64 running sums' registers for the
  // stage loop; otherwise they accumulate in registers and are stored once.
  const int64_t go = i0 + drow;
  double* const Yb = reinterpret_cast<double*>(Y + it.ybase + (int64_t)blockIdx.z * pstride);
  const int cb = (dq % DPC) * DC;
  auto yidx = [&](int c) { return 2 * (go + (it.ycol + cb + c) * ldy) + dq / DPC; };
#if OZ_GACC
  double* yacc = nullptr;
#else
  double yacc[DC];
#pragma unroll
  for (int c = 0; c < DC; ++c) yacc[c] = 0.0;
#endif
  uint32_t amp_hi = 0;  // max high word of the scaled amplitudes
  if (OZ_ZERO_ACC) {  // every warp zeroes the accumulator columns it drains
#pragma unroll
    for (int j = 0; j < OZ_NDIAG; ++j) tmem_zero<DC>(tmem + ((uint32_t)((warp & 3) * 32) << 16) + j * Z::BN2 + dq * DC);
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  }

  auto drain = [&](int d) {
    OZT_BEGIN(t4)
    mbar_wait(acc_full, (uint32_t)d & 1u);
    if (lane == 0) { OZT_END(t4, 4) }
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    double t[DC];
#pragma unroll
    for (int j = OZ_NDIAG - 1; j >= 0; --j) {
      const uint32_t base = tmem + ((uint32_t)((warp & 3) * 32) << 16) + j * Z::BN2 + dq * DC;
      uint32_t v[DC];
      if constexpr (DC % 16 == 0) {
#pragma unroll
        for (int q = 0; q < DC / 16; ++q) {
          uint32_t w[16];
          tmem_ld16(base + 16 * q, w);
#pragma unroll
          for (int u = 0; u < 16; ++u) v[16 * q + u] = w[u];
        }
      } else {
#pragma unroll
        for (int q = 0; q < DC / 4; ++q) {
          uint32_t w[4];
          tmem_ld4(base + 4 * q, w);
#pragma unroll
          for (int u = 0; u < 4; ++u) v[4 * q + u] = w[u];
        }
      }
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
      if (OZ_ZERO_ACC) tmem_zero<DC>(base);  // the next chunk's MMAs all accumulate
#pragma unroll
      for (int c = 0; c < DC; ++c) t[c] = (j == OZ_NDIAG - 1) ? i2d(v[c]) : fma(t[c], 256.0, i2d(v[c]));
    }
    if (OZ_ZERO_ACC) asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    const int S = Srow[(d & 1) * OZ_BM + drow];
    const int c0 = cb;
#if OZ_GACC
    if (go < m_out) {
#pragma unroll
      for (int c = 0; c < DC; ++c)
        if (cb + c < it.ncols) {
          const double v = t[c] * pow2(8 * OZ_E0 - S - Ts[c0 + c]);
          Yb[yidx(c)] = d == 0 ? v : Yb[yidx(c)] + v;
        }
    }
    (void)yacc;
#else
#pragma unroll
    for (int c = 0; c < DC; ++c) yacc[c] = fma(t[c], pow2(8 * OZ_E0 - S - Ts[c0 + c]), yacc[c]);
#endif
  };

  // All MMAs of a stage, issued by one converged warp (the group's last to
  // write it): the base descriptors are warp-uniform values and every MMA adds
  // a compile-time offset, so the descriptor math stays in uniform registers
  // and one elected lane issues each tcgen05.mma back to back (round 1 issued
  // from a divergent lane: ~100 cycles of R2UR / branch loops per MMA, which
  // starved the tensor pipe on the small N = 64 MMAs).
  auto issue_stage = [&](int slot_in, uint32_t ph, int s, int nst) {
    const uint32_t slot = warp_uniform((uint32_t)slot_in);
    mbar_wait(fullB(slot), ph);
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tm = warp_uniform(tmem);
    const uint64_t da0 = smem_desc(warp_uniform(sA) + slot * OZ_ASTAGE, OZ_AHALF, 128);
    const uint64_t db0 = smem_desc(warp_uniform(sB) + slot * Z::BSTAGE, (Z::BROWS / 8) * 128, 128);
    const bool first = s == 0;
    constexpr OzSched kS = make_sched(Z::MAXB);
#pragma unroll
    for (int i = 0; i < kS.n; ++i) {
      const uint32_t e = kS.code[i];
      const int h = e & 1, p = (e >> 1) & 7, jlo = (e >> 4) & 15, nb = (e >> 8) & 31;
      const bool init = (e >> 13) & 1;
      const int q0 = jlo + OZ_E0 - p;
      // descriptor address fields hold addr >> 4 (14 bits; shared addresses < 2^18): offsets add in place
      const uint64_t da = da0 + (uint64_t)(((h * OZ_NSL + p) * OZ_ABLK) >> 4);
      const uint64_t db = db0 + (uint64_t)((h * Z::BOPER + q0 * Z::BN2 * 16) >> 4);
#ifdef OZ_TRACE
      if (g_oz_mode & 1) continue;
#endif
      if (!(OZ_EXP & 1) && elect_one())  // experiment bit 1: no MMAs
        mma_i8(tm + jlo * Z::BN2, da, db, idesc_i8(128, nb * Z::BN2, p == OZ_NSL - 1, true), (init && first) ? 0u : 1u);
    }
    if (elect_one()) {
      mma_commit(empty(slot));
      if (s == nst - 1) mma_commit(acc_full);
    }
    __syncwarp();
  };

  // The last warp to finish stage g issues its MMAs only after evaluating its
  // entries of stage g+1: FP64 and tensor work time-share the datapath, so
  // the tensor then runs during the integer write phase (transposes, shared
  // stores) instead of blocking the next evaluation.  Ordering holds: the
  // issuer writes stage g+1 only after issuing stage g.
  int pend_slot = -1, pend_s = 0, pend_nst = 0;
  uint32_t pend_ph = 0;
  int g = 0;
  for (int d = 0; d < nchunks; ++d) {
    const int64_t c0 = kb + (int64_t)d * Z::KD;
    const int npts = (int)min((int64_t)Z::KD, ke - c0);
    const int nst = (int)ceil_div((int64_t)npts, (int64_t)OZ_KS);
    // ---- chunk setup: input points, per-row scale S (bound on |a| over the chunk)
    OZT_BEGIN(t6)
    __syncthreads();  // previous chunk's points no longer read
    const int64_t p0 = it.row0 + c0;
    const double bx = inp.x[p0];
    const double by = KIND == KK_NUFFT ? 0.0 : inp.y[p0];
    const double bz = KIND == KK_PLATES ? inp.z[p0] : 0.0;
    for (int k = tid; k < nst * OZ_KS; k += OZS_THREADS) {
      // entries past the chunk repeat its first point: finite values whose B rows are zero
      const int64_t pk = p0 + (k < npts ? k : 0);
      const double x = inp.x[pk];
      const double y = KIND == KK_NUFFT ? 0.0 : inp.y[pk];
      const double z = KIND == KK_PLATES ? inp.z[pk] : 0.0;
      PD[k] = make_double2(x, y);
      if (KIND == KK_PLATES) PZ[k] = z;
    }
    if (tid < OZ_BM) Smin[tid] = 0x7F7FFFFFu;  // FLT_MAX bits
    __syncthreads();
    if (KIND != KK_NUFFT) {
      // bounding boxes of the sub-boxes of 32 consecutive (tree-ordered) points,
      // in float coordinates local to the chunk's first point
      float4* BX = reinterpret_cast<float4*>(smem + Z::SM_BOX);  // [NBOX][lo, hi]
#pragma unroll
      for (int q = 0; q < Z::NBOX / OZS_WARPS; ++q) {
        const int sb = warp * (Z::NBOX / OZS_WARPS) + q;
        const int k = min(sb * 32 + lane, Z::KD - 1);
        const double2 pd = PD[k];
        const float px = (float)(pd.x - bx), py = (float)(pd.y - by);
        const float pz = KIND == KK_PLATES ? (float)(PZ[k] - bz) : 0.f;
        float lx = px, ly = py, lz = pz, hx = px, hy = py, hz = pz;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
          lx = fminf(lx, __shfl_xor_sync(0xffffffffu, lx, o));
          ly = fminf(ly, __shfl_xor_sync(0xffffffffu, ly, o));
          lz = fminf(lz, __shfl_xor_sync(0xffffffffu, lz, o));
          hx = fmaxf(hx, __shfl_xor_sync(0xffffffffu, hx, o));
          hy = fmaxf(hy, __shfl_xor_sync(0xffffffffu, hy, o));
          hz = fmaxf(hz, __shfl_xor_sync(0xffffffffu, hz, o));
        }
        if (lane == 0) {
          BX[2 * sb] = make_float4(lx, ly, lz, 0.f);
          BX[2 * sb + 1] = make_float4(hx, hy, hz, 0.f);
        }
      }
      __syncthreads();
      // per row: min squared distance to the boxes (a lower bound of the
      // distance to every point); exact over a box's points only when the row
      // point lies inside it
      const int r = tid & (OZ_BM - 1), part = tid >> 7;
      const int64_t gr = min(i0 + r, m_out - 1);
      const float lx = (float)(outp.x[gr] - bx), ly = (float)(outp.y[gr] - by);
      const float lz = KIND == KK_PLATES ? (float)(outp.z[gr] - bz) : 0.f;
      const int nbox = (nst * OZ_KS) / 32;
      float mn = 3.0e38f;
      for (int b = part; b < nbox; b += OZS_THREADS / OZ_BM) {
        const float4 lo = BX[2 * b], hi = BX[2 * b + 1];
        const float dx = fmaxf(fmaxf(lo.x - lx, lx - hi.x), 0.f);
        const float dy = fmaxf(fmaxf(lo.y - ly, ly - hi.y), 0.f);
        const float dz = KIND == KK_PLATES ? fmaxf(fmaxf(lo.z - lz, lz - hi.z), 0.f) : 0.f;
        float d2 = fmaf(dz, dz, fmaf(dy, dy, dx * dx));
        if (d2 == 0.f) {
          d2 = 3.0e38f;
          for (int k = b * 32; k < b * 32 + 32; ++k) {
            const double2 pd = PD[k];
            const float ex = lx - (float)(pd.x - bx), ey = ly - (float)(pd.y - by);
            float e2 = fmaf(ex, ex, ey * ey);
            if (KIND == KK_PLATES) {
              const float ez = lz - (float)(PZ[k] - bz);
              e2 = fmaf(ez, ez, e2);
            }
            d2 = fminf(d2, e2);
          }
        }
        mn = fminf(mn, d2);
      }
      atomicMin(&Smin[r], __float_as_uint(mn));
    }
    __syncthreads();
    if (tid < OZ_BM) {
      int S = OZ_ABITS - 1;  // NUFFT: |a| = 1
      if (KIND != KK_NUFFT) {
        const float mn = __uint_as_float(Smin[tid]);
        // amplitude bound with a factor-2 margin for the float distance estimate
        double amax = mn > 1e-36f ? 2.0 / sqrt((double)mn) : 1e300;
        if (KIND == KK_PLATES) amax /= keval::kFourPi;
        S = amax < 1e300 ? (OZ_ABITS - 1) - ilogb(amax) : 0;
      }
      Srow[(d & 1) * OZ_BM + tid] = S;
    }
    __syncthreads();
    if (lane == 0) { OZT_END(t6, 6) }
    // row scale 2^S, folded with the amplitude constant (see entry_rounded)
    const double p2 = pow2(Srow[(d & 1) * OZ_BM + erow]);  // NUFFT row scale
    const int es = (Srow[(d & 1) * OZ_BM + erow] + 1) << 20;  // Helmholtz: 2h 2^S, as an exponent add
    for (int s = 0; s < nst; ++s, ++g) {
      const int slot = g % OZ_NST;
      const uint32_t ph = (uint32_t)(g / OZ_NST) & 1u;
      const int64_t k0 = c0 + (int64_t)s * OZ_KS;  // item-relative first entry of the stage
      // ring slot: free once the MMAs of stage g - 2 completed; then its B
      // image is refilled (waiting after the evaluation instead measured 5 %
      // slower: the B copy then lands too late for the stage's MMAs)
      OZT_BEGIN(t3)
      if (g >= OZ_NST) mbar_wait(empty(slot), ph ^ 1u);
      if (lane == 0) { OZT_END(t3, 3) }
      if (tid == 0) {
        if (OZ_EXP & 4) {  // experiment: no B refill (the slot's image stays)
          asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" ::"r"(fullB(slot)) : "memory");
        } else {
          mbar_expect_tx(fullB(slot), Z::BSTAGE);
          bulk_g2s(sB + slot * Z::BSTAGE, bimg + (it.bstage0 + k0 / OZ_KS) * (int64_t)Z::BSTAGE, Z::BSTAGE,
                   fullB(slot));
        }
      }
      // ---- evaluate 8 entries, scale, round (magic-number: low word = low
      // 32 bits of the integer, high word - 0x43380000 = high 32 bits)
      uint32_t lo_r[OZS_EPT], hi_r[OZS_EPT], lo_i[OZS_EPT], hi_i[OZS_EPT];
      const int kl = s * OZ_KS + kofs;  // chunk-relative
      OZT_BEGIN(t0)
#pragma unroll
      for (int e = 0; e < OZS_EPT; ++e) {
        const double2 sp = PD[kl + e];
        const double sz = KIND == KK_PLATES ? PZ[kl + e] : 0.0;
        double tr, ti, amp;
        if (OZ_EXP & 2) {  // experiment: no evaluation (cheap data-dependent integers)
          tr = keval::kMagic + (double)(kl + e) + sp.x;
          ti = keval::kMagic - (double)(kl + e);
          amp = 0.0;
        } else if (MODE == OP_N)
          entry_rounded<KIND, false>(ox, oy, oz, sp.x, sp.y, sz, kappa, p2, es, tab, tr, ti, amp);
        else
          entry_rounded<KIND, MODE == OP_H>(sp.x, sp.y, sz, ox, oy, oz, kappa, p2, es, tab, tr, ti, amp);
        amp_hi = max(amp_hi, (uint32_t)__double2hiint(amp));
        lo_r[e] = (uint32_t)__double2loint(tr);
        hi_r[e] = (uint32_t)__double2hiint(tr) - 0x43380000u;
        lo_i[e] = (uint32_t)__double2loint(ti);
        hi_i[e] = (uint32_t)__double2hiint(ti) - 0x43380000u;
      }
#ifdef OZ_TRACE
      {
        uint32_t dep = 0;
#pragma unroll
        for (int e = 0; e < 8; ++e) dep ^= lo_r[e] ^ hi_r[e] ^ lo_i[e] ^ hi_i[e];
        if (dep == 0x12345678u) amp_hi ^= 1u;
      }
#endif
      if (lane == 0) { OZT_END(t0, 0) }
      if (pend_slot >= 0) {  // the last stage's issuing warp (converged)
        OZT_BEGIN(t2)
        issue_stage(pend_slot, pend_ph, pend_s, pend_nst);
        if (lane == 0) { OZT_END(t2, 2) }
        pend_slot = -1;
      }
      OZT_BEGIN(t1)
      // ---- byte slices -> canonical K-major A images (4x4 byte transposes)
      uint8_t* a0 = smem + Z::SM_A + slot * OZ_ASTAGE;
      const int off = (kofs >> 4) * OZ_AHALF + (erow >> 3) * 128 + (erow & 7) * 16 + (kofs & 15);
#pragma unroll
      for (int h = 0; h < ((OZ_EXP & 8) ? 0 : 2); ++h) {  // experiment bit 3: no A writes
#pragma unroll
        for (int gq = 0; gq < OZS_EPT / 8; ++gq) {  // groups of 8 entries = 8 bytes per slice
          const uint32_t* lo = (h ? lo_i : lo_r) + 8 * gq;
          const uint32_t* hi = (h ? hi_i : hi_r) + 8 * gq;
          uint32_t l0[4], l1[4], h0[4], h1[4];
          transpose4(lo[0], lo[1], lo[2], lo[3], l0);
          transpose4(lo[4], lo[5], lo[6], lo[7], l1);
          transpose4(hi[0], hi[1], hi[2], hi[3], h0);
          transpose4(hi[4], hi[5], hi[6], hi[7], h1);
          uint8_t* pl = a0 + h * OZ_NSL * OZ_ABLK + off + 8 * gq;
#pragma unroll
          for (int p = 0; p < 4; ++p) *reinterpret_cast<uint2*>(pl + p * OZ_ABLK) = make_uint2(l0[p], l1[p]);
#pragma unroll
          for (int p = 0; p < OZ_NSL - 4; ++p)
            *reinterpret_cast<uint2*>(pl + (4 + p) * OZ_ABLK) = make_uint2(h0[p], h1[p]);
        }
      }
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      if (lane == 0) { OZT_END(t1, 1) }
      if (s == 0 && d > 0) drain(d - 1);  // TMEM must be free before this stage's MMAs
      asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
      __syncwarp();
      unsigned last = 0;
      if (lane == 0) {
        __threadfence_block();
        last = atomicAdd(&cnt[slot], 1u) == OZS_WARPS - 1;  // last warp in: issues the stage (deferred)
        if (last) {
          cnt[slot] = 0;
          __threadfence_block();
        }
      }
      if (__shfl_sync(0xffffffffu, last, 0)) {
        pend_slot = slot;
        pend_ph = ph;
        pend_s = s;
        pend_nst = nst;
        if (!OZ_DEFER) {  // experiment: issue at once (lockstep)
          issue_stage(pend_slot, pend_ph, pend_s, pend_nst);
          pend_slot = -1;
        }
      }
      __syncwarp();
    }
  }
  if (pend_slot >= 0) issue_stage(pend_slot, pend_ph, pend_s, pend_nst);
  __syncwarp();
  if (nchunks > 0) drain(nchunks - 1);
  if (KIND != KK_NUFFT && amp_hi >= amp_limit_hi<KIND>()) atomicOr(flag, 2);

  // ---- store (OZ_GACC: only an empty input range has not written its zeros)
  if (go < m_out && (!OZ_GACC || nchunks == 0)) {
#pragma unroll
    for (int c = 0; c < DC; ++c)
      if (cb + c < it.ncols) Yb[yidx(c)] = OZ_GACC ? 0.0 : yacc[c];
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (tid == 0) { OZT_END(t5, 5) }
  if (warp == 0) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(Z::TMEM_COLS));
  }
}

// ------------------------------------------------------- K2, CTA pairs
// Probe tiles of 33..40 columns (config 2's fused leaf rounds, 6 + 10 + 18 =
// 34; config 1's 34..40-wide levels) need 7 x 80 = 560 accumulator columns,
// more than TMEM holds, so one CTA cannot take them in one pass; two passes
// evaluate every kernel entry twice.  A cluster of two CTAs on the same 128
// output rows and input range instead evaluates each stage ONCE: CTA r
// evaluates the stage's K-half r (16 of the 32 input entries) and sends its
// 24 KB of A slices to the peer with one DSMEM bulk copy (async proxy,
// completing on the peer's fullA barrier), and the pair splits the diagonal
// blocks: CTA 0 keeps e = 4, 5, 9, 10 (14 slice pairs, 4 x 80 TMEM columns),
// CTA 1 e = 6, 7, 8 (12 pairs, 3 x 80).  Each CTA drains its own diagonals
// into its own partial output slice; the split-K reduce adds the two.
// A stage layout here: [K-half][plane][slice] 2 KB blocks, so a CTA's half is
// one contiguous 24 KB (the MMA descriptor's K step LBO = 24 KB).
// The ring slot's `empty` barrier counts BOTH CTAs' MMA commits (multicast):
// a CTA overwrites its half -- in its own slot and, by the copy, in the
// peer's -- only when both have finished reading the stage two back.
#ifndef OZP_EW
#define OZP_EW 16
#endif
constexpr int OZP_WARPS = OZP_EW;                       // evaluation warps per CTA of a pair
constexpr int OZP_THREADS = OZP_WARPS * 32;
constexpr int OZP_EPT = OZ_BM * (OZ_KS / 2) / OZP_THREADS;  // entries per thread per stage: 4 or 8
static_assert(OZP_EPT == 4 || OZP_EPT == 8, "pair thread mapping");
constexpr int OZP_NCB = 40;   // pair tile: 33..40 columns
constexpr int OZP_NCB48 = 48; // 41..48 columns, 3D plates only (its 1024-entry chunks leave the smem room)
constexpr int OZP_HALF = OZ_AHALF;  // 24 KB: one CTA's K-half of a stage
static_assert(OZ_E0 == 4 && OZ_NDIAG == 7, "pair diagonal split assumes e = 4 .. 10");
__host__ __device__ constexpr int ozp_nloc(int cr) { return cr == 0 ? 4 : 3; }
// global diagonal block of local block jl
__host__ __device__ constexpr int ozp_glob(int cr, int jl) { return cr == 0 ? (jl < 2 ? jl : jl + 3) : jl + 2; }
// local block of global block j, or -1
__host__ __device__ constexpr int ozp_loc(int cr, int j) {
  return cr == 0 ? (j < 2 ? j : (j >= 5 ? j - 3 : -1)) : ((j >= 2 && j <= 4) ? j - 2 : -1);
}
// schedule of CTA cr: per plane and slice, maximal runs of its blocks (contiguous
// locally AND globally), windows of <= maxb blocks.  packed as mma_code plus the
// local first block at bit 14
constexpr OzSched make_sched_pair(int cr, int maxb) {
  OzSched sc{};
  sc.n = 0;
  constexpr int T = OZ_NSL - 1, D = OZ_NDIAG;
  for (int h = 0; h < 2; ++h)
    for (int p = T; p >= 0; --p) {
      const int jlo = p > OZ_E0 ? p - OZ_E0 : 0;
      const int jhi = (D - 1) < (T + p - OZ_E0) ? (D - 1) : (T + p - OZ_E0);
      int j = jlo;
      while (j <= jhi) {
        if (ozp_loc(cr, j) < 0) { ++j; continue; }
        int e = j;
        while (e + 1 <= jhi && ozp_loc(cr, e + 1) == ozp_loc(cr, e) + 1 && e + 1 - j < maxb) ++e;
        sc.code[sc.n++] = mma_code(h, p, j, e - j + 1, 0) | ((uint32_t)ozp_loc(cr, j) << 14);
        j = e + 1;
      }
    }
  return sc;
}
template <int CR, int NCB>
struct OzPairSched {
  static constexpr OzSched value = make_sched_pair(CR, OzT<NCB, 1024, false>::MAXB);
};
__device__ __forceinline__ uint32_t cluster_ctarank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ uint32_t mapa_peer(uint32_t addr, uint32_t peer) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(addr), "r"(peer));
  return r;
}
// tcgen05.commit arriving on the barrier at this offset in both CTAs of the pair
__device__ __forceinline__ void mma_commit_pair(uint32_t bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
                   bar),
               "h"((uint16_t)3)
               : "memory");
}
// local shared -> peer shared bulk copy, completing transaction bytes on the peer's barrier
__device__ __forceinline__ void bulk_s2peer(uint32_t dst_cluster, uint32_t src, uint32_t bytes, uint32_t bar_cluster) {
  asm volatile("cp.async.bulk.shared::cluster.shared::cta.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   dst_cluster),
               "r"(src), "r"(bytes), "r"(bar_cluster)
               : "memory");
}

template <int KIND, int MODE, int NCB>
__global__ void __launch_bounds__(OZP_THREADS, 1)
    matvec_oz_pair_kernel(Points outp, Points inp, double kappa, int64_t m_out, const uint8_t* __restrict__ bimg,
                          const int32_t* __restrict__ Tg, double2* __restrict__ Y, int64_t ldy,
                          const OzItem* __restrict__ items, int64_t rows_per_split, int64_t pstride,
                          int* __restrict__ flag) {
  using Z = OzT<NCB, oz_kd(KIND), KIND == KK_PLATES>;
  extern __shared__ __align__(1024) uint8_t smem[];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const uint32_t cr = cluster_ctarank(), peer = cr ^ 1u;
  const OzItem it = items[blockIdx.y];
  const int64_t i0 = (int64_t)(blockIdx.x >> 1) * OZ_BM;
  const int64_t kb = (int64_t)blockIdx.z * rows_per_split;
  const int64_t ke = min(it.rows, kb + rows_per_split);
  const int64_t nk = ke > kb ? ke - kb : 0;
  const int nchunks = (int)ceil_div(nk, (int64_t)Z::KD);

  double2* PD = reinterpret_cast<double2*>(smem + Z::SM_PD);
  double* PZ = reinterpret_cast<double*>(smem + Z::SM_PZ);
  int* Srow = reinterpret_cast<int*>(smem + Z::SM_S);
  int* Ts = reinterpret_cast<int*>(smem + Z::SM_T);
  unsigned* Smin = reinterpret_cast<unsigned*>(smem + Z::SM_MIN);
  unsigned* cnt = reinterpret_cast<unsigned*>(smem + Z::SM_CNT);
  const uint32_t bar0 = smem_u32(smem + Z::SM_BAR);
  auto fullB = [&](int s) { return bar0 + 8u * s; };
  auto empty = [&](int s) { return bar0 + 8u * (OZ_NST + s); };
  const uint32_t acc_full = bar0 + 8u * (2 * OZ_NST);
  auto fullA = [&](int s) { return bar0 + 8u * (2 * OZ_NST + 1 + s); };  // the peer's K-half landed
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + Z::SM_TMEM);
  constexpr int COLS0 = pow2_ceil(ozp_nloc(0) * Z::BN2), COLS1 = pow2_ceil(ozp_nloc(1) * Z::BN2);

  if (warp == 0) {
    if (cr == 0)
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                   "n"(COLS0));
    else
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                   "n"(COLS1));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 32) {
    for (int s = 0; s < OZ_NST; ++s) {
      mbar_init(fullB(s), 1);
      mbar_init(empty(s), 2);  // this CTA's and the peer's MMA commits
      mbar_init(fullA(s), 1);
      cnt[s] = 0;
    }
    mbar_init(acc_full, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (tid < NCB) Ts[tid] = Tg[blockIdx.y * OZ_MAXCB + tid];
  double2* tab = reinterpret_cast<double2*>(smem + Z::SM_TAB);
  for (int j = tid; j < keval::kTabN; j += OZP_THREADS) {  // plates: times 1/(4 pi)
    const double2 t = g_oz_tab[j];
    tab[j] = KIND == KK_PLATES ? make_double2(t.x * (1.0 / keval::kFourPi), t.y * (1.0 / keval::kFourPi)) : t;
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  cluster_sync_all();  // barriers of both CTAs initialised before any remote arrive
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = *tmem_slot;
  const uint32_t sA = smem_u32(smem + Z::SM_A), sB = smem_u32(smem + Z::SM_B);

  // evaluation: 16 warps: row warp * 8 + lane / 4, entries 4 (lane & 3) .. + 3
  // of this CTA's K-half; 8 warps: row warp * 16 + lane / 2, entries 8 (lane & 1) .. + 7
  const int erow = OZP_EPT == 4 ? warp * 8 + (lane >> 2) : warp * 16 + (lane >> 1);
  const int kq = OZP_EPT == 4 ? (lane & 3) * 4 : (lane & 1) * 8;
  const int64_t gi = min(i0 + erow, m_out - 1);
  const double ox = outp.x[gi];
  const double oy = KIND == KK_NUFFT ? 0.0 : outp.y[gi];
  const double oz = KIND == KK_PLATES ? outp.z[gi] : 0.0;
  // drain: TMEM lane quarter = warp & 3, column quarter = warp >> 2 of [Re y | Im y]
  const int drow = (warp & 3) * 32 + lane;
  const int dq = warp >> 2;
  constexpr int DC = OZP_WARPS == 16 ? Z::DC : NCB;  // drained columns per thread
  constexpr int DPC = NCB / DC;
  const int nloc = ozp_nloc((int)cr);
  const int64_t go = i0 + drow;
  // this CTA's partial output slice (the split-K reduce adds the pair's two)
  double* const Yb = reinterpret_cast<double*>(Y + it.ybase + ((int64_t)blockIdx.z * 2 + cr) * pstride);
  const int cb = (dq % DPC) * DC;
  auto yidx = [&](int c) { return 2 * (go + (it.ycol + cb + c) * ldy) + dq / DPC; };
  uint32_t amp_hi = 0;
  for (int jl = 0; jl < nloc; ++jl) tmem_zero<DC>(tmem + ((uint32_t)((warp & 3) * 32) << 16) + jl * Z::BN2 + dq * DC);
  asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");

  auto drain = [&](int d) {
    mbar_wait(acc_full, (uint32_t)d & 1u);
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    // partial Horner over this CTA's diagonals, in global diagonal order
    double t[DC];
#pragma unroll
    for (int c = 0; c < DC; ++c) t[c] = 0.0;
    int jprev = -1;
    for (int jl = nloc - 1; jl >= 0; --jl) {
      const int j = ozp_glob((int)cr, jl);
      const uint32_t base = tmem + ((uint32_t)((warp & 3) * 32) << 16) + jl * Z::BN2 + dq * DC;
      uint32_t v[DC];
#pragma unroll
      for (int q = 0; q < DC / 4; ++q) {
        uint32_t w[4];
        tmem_ld4(base + 4 * q, w);
#pragma unroll
        for (int u = 0; u < 4; ++u) v[4 * q + u] = w[u];
      }
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
      tmem_zero<DC>(base);
      const double sh = jprev < 0 ? 0.0 : pow2(8 * (jprev - j));  // exact: 2^8 steps
#pragma unroll
      for (int c = 0; c < DC; ++c) t[c] = fma(t[c], sh, i2d(v[c]));
      jprev = j;
    }
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    // t holds sum_j d_j 2^{8 (j - jmin)}; jmin = the lowest global block of this CTA
    const int jmin = jprev;
    const int S = Srow[(d & 1) * OZ_BM + drow];
    const int c0 = cb;
    if (go < m_out) {
#pragma unroll
      for (int c = 0; c < DC; ++c)
        if (cb + c < it.ncols) {
          const double v = t[c] * pow2(8 * (OZ_E0 + jmin) - S - Ts[c0 + c]);
          Yb[yidx(c)] = d == 0 ? v : Yb[yidx(c)] + v;
        }
    }
  };

  auto issue_stage = [&](int slot_in, uint32_t ph, int s, int nst) {
    const uint32_t slot = warp_uniform((uint32_t)slot_in);
    mbar_wait(fullB(slot), ph);
    mbar_wait(fullA(slot), ph);
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tm = warp_uniform(tmem);
    // A: K step = the other CTA's half (LBO 24 KB), 8-row groups 128 B apart
    const uint64_t da0 = smem_desc(warp_uniform(sA) + slot * OZ_ASTAGE, OZP_HALF, 128);
    const uint64_t db0 = smem_desc(warp_uniform(sB) + slot * Z::BSTAGE, (Z::BROWS / 8) * 128, 128);
    auto run = [&](auto sched) {
      constexpr OzSched kS = decltype(sched)::value;
      (void)sched;
#pragma unroll
      for (int i = 0; i < kS.n; ++i) {
        const uint32_t e = kS.code[i];
        const int h = e & 1, p = (e >> 1) & 7, jlo = (e >> 4) & 15, nb = (e >> 8) & 31, jl = (e >> 14) & 15;
        const int q0 = jlo + OZ_E0 - p;
        const uint64_t da = da0 + (uint64_t)(((h * OZ_NSL + p) * (OZP_HALF / OZ_NSL / 2)) >> 4);
        const uint64_t db = db0 + (uint64_t)((h * Z::BOPER + q0 * Z::BN2 * 16) >> 4);
        if (elect_one()) mma_i8(tm + jl * Z::BN2, da, db, idesc_i8(128, nb * Z::BN2, p == OZ_NSL - 1, true), 1u);
      }
    };
    if (cr == 0)
      run(OzPairSched<0, NCB>{});
    else
      run(OzPairSched<1, NCB>{});
    if (elect_one()) {
      mma_commit_pair(empty(slot));
      if (s == nst - 1) mma_commit(acc_full);
    }
    __syncwarp();
  };

  int pend_slot = -1, pend_s = 0, pend_nst = 0;
  uint32_t pend_ph = 0;
  int g = 0;
  for (int d = 0; d < nchunks; ++d) {
    const int64_t c0 = kb + (int64_t)d * Z::KD;
    const int npts = (int)min((int64_t)Z::KD, ke - c0);
    const int nst = (int)ceil_div((int64_t)npts, (int64_t)OZ_KS);
    // ---- chunk setup (both CTAs compute the same row scales S)
    __syncthreads();
    const int64_t p0 = it.row0 + c0;
    const double bx = inp.x[p0];
    const double by = KIND == KK_NUFFT ? 0.0 : inp.y[p0];
    const double bz = KIND == KK_PLATES ? inp.z[p0] : 0.0;
    for (int k = tid; k < nst * OZ_KS; k += OZP_THREADS) {
      const int64_t pk = p0 + (k < npts ? k : 0);
      PD[k] = make_double2(inp.x[pk], KIND == KK_NUFFT ? 0.0 : inp.y[pk]);
      if (KIND == KK_PLATES) PZ[k] = inp.z[pk];
    }
    if (tid < OZ_BM) Smin[tid] = 0x7F7FFFFFu;
    __syncthreads();
    if (KIND != KK_NUFFT) {
      float4* BX = reinterpret_cast<float4*>(smem + Z::SM_BOX);
#pragma unroll
      for (int q = 0; q < Z::NBOX / OZP_WARPS; ++q) {
        const int sb = warp * (Z::NBOX / OZP_WARPS) + q;
        const int k = min(sb * 32 + lane, Z::KD - 1);
        const double2 pd = PD[k];
        const float px = (float)(pd.x - bx), py = (float)(pd.y - by);
        const float pz = KIND == KK_PLATES ? (float)(PZ[k] - bz) : 0.f;
        float lx = px, ly = py, lz = pz, hx = px, hy = py, hz = pz;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
          lx = fminf(lx, __shfl_xor_sync(0xffffffffu, lx, o));
          ly = fminf(ly, __shfl_xor_sync(0xffffffffu, ly, o));
          lz = fminf(lz, __shfl_xor_sync(0xffffffffu, lz, o));
          hx = fmaxf(hx, __shfl_xor_sync(0xffffffffu, hx, o));
          hy = fmaxf(hy, __shfl_xor_sync(0xffffffffu, hy, o));
          hz = fmaxf(hz, __shfl_xor_sync(0xffffffffu, hz, o));
        }
        if (lane == 0) {
          BX[2 * sb] = make_float4(lx, ly, lz, 0.f);
          BX[2 * sb + 1] = make_float4(hx, hy, hz, 0.f);
        }
      }
      __syncthreads();
      const int r = tid & (OZ_BM - 1), part = tid >> 7;
      const int64_t gr = min(i0 + r, m_out - 1);
      const float lx = (float)(outp.x[gr] - bx), ly = (float)(outp.y[gr] - by);
      const float lz = KIND == KK_PLATES ? (float)(outp.z[gr] - bz) : 0.f;
      const int nbox = (nst * OZ_KS) / 32;
      float mn = 3.0e38f;
      for (int b = part; b < nbox; b += OZP_THREADS / OZ_BM) {
        const float4 lo = BX[2 * b], hi = BX[2 * b + 1];
        const float dx = fmaxf(fmaxf(lo.x - lx, lx - hi.x), 0.f);
        const float dy = fmaxf(fmaxf(lo.y - ly, ly - hi.y), 0.f);
        const float dz = KIND == KK_PLATES ? fmaxf(fmaxf(lo.z - lz, lz - hi.z), 0.f) : 0.f;
        float d2 = fmaf(dz, dz, fmaf(dy, dy, dx * dx));
        if (d2 == 0.f) {
          d2 = 3.0e38f;
          for (int k = b * 32; k < b * 32 + 32; ++k) {
            const double2 pd = PD[k];
            const float ex = lx - (float)(pd.x - bx), ey = ly - (float)(pd.y - by);
            float e2 = fmaf(ex, ex, ey * ey);
            if (KIND == KK_PLATES) {
              const float ez = lz - (float)(PZ[k] - bz);
              e2 = fmaf(ez, ez, e2);
            }
            d2 = fminf(d2, e2);
          }
        }
        mn = fminf(mn, d2);
      }
      atomicMin(&Smin[r], __float_as_uint(mn));
    }
    __syncthreads();
    if (tid < OZ_BM) {
      int S = OZ_ABITS - 1;
      if (KIND != KK_NUFFT) {
        const float mn = __uint_as_float(Smin[tid]);
        double amax = mn > 1e-36f ? 2.0 / sqrt((double)mn) : 1e300;
        if (KIND == KK_PLATES) amax /= keval::kFourPi;
        S = amax < 1e300 ? (OZ_ABITS - 1) - ilogb(amax) : 0;
      }
      Srow[(d & 1) * OZ_BM + tid] = S;
    }
    __syncthreads();
    const double p2 = pow2(Srow[(d & 1) * OZ_BM + erow]);  // NUFFT row scale
    const int es = (Srow[(d & 1) * OZ_BM + erow] + 1) << 20;  // Helmholtz: 2h 2^S, as an exponent add
    for (int s = 0; s < nst; ++s, ++g) {
      const int slot = g % OZ_NST;
      const uint32_t ph = (uint32_t)(g / OZ_NST) & 1u;
      const int64_t k0 = c0 + (int64_t)s * OZ_KS;
      // slot free: both CTAs' MMAs of stage g - 2 done
      if (g >= OZ_NST) mbar_wait(empty(slot), ph ^ 1u);
      if (tid == 0) {
        mbar_expect_tx(fullB(slot), Z::BSTAGE);
        bulk_g2s(sB + slot * Z::BSTAGE, bimg + (it.bstage0 + k0 / OZ_KS) * (int64_t)Z::BSTAGE, Z::BSTAGE, fullB(slot));
        if (OZ_EXP & 16)  // experiment: no DSMEM exchange (wrong results)
          asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" ::"r"(fullA(slot)) : "memory");
        else
          mbar_expect_tx(fullA(slot), OZP_HALF);  // the peer's half of this stage
      }
      // ---- evaluate this CTA's 4 entries of its K-half
      uint32_t lo_r[OZP_EPT], hi_r[OZP_EPT], lo_i[OZP_EPT], hi_i[OZP_EPT];
      const int kl = s * OZ_KS + (int)cr * 16 + kq;  // chunk-relative
#pragma unroll
      for (int e = 0; e < OZP_EPT; ++e) {
        const double2 sp = PD[kl + e];
        const double sz = KIND == KK_PLATES ? PZ[kl + e] : 0.0;
        double tr, ti, amp;
        if (MODE == OP_N)
          entry_rounded<KIND, false>(ox, oy, oz, sp.x, sp.y, sz, kappa, p2, es, tab, tr, ti, amp);
        else
          entry_rounded<KIND, MODE == OP_H>(sp.x, sp.y, sz, ox, oy, oz, kappa, p2, es, tab, tr, ti, amp);
        amp_hi = max(amp_hi, (uint32_t)__double2hiint(amp));
        lo_r[e] = (uint32_t)__double2loint(tr);
        hi_r[e] = (uint32_t)__double2hiint(tr) - 0x43380000u;
        lo_i[e] = (uint32_t)__double2loint(ti);
        hi_i[e] = (uint32_t)__double2hiint(ti) - 0x43380000u;
      }
      if (pend_slot >= 0) {
        issue_stage(pend_slot, pend_ph, pend_s, pend_nst);
        pend_slot = -1;
      }
      // ---- byte slices -> this CTA's K-half of the A images: [plane][slice] 2 KB blocks
      uint8_t* a0 = smem + Z::SM_A + slot * OZ_ASTAGE + cr * OZP_HALF;
      const int off = (erow >> 3) * 128 + (erow & 7) * 16 + kq;
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const uint32_t* lo = h ? lo_i : lo_r;
        const uint32_t* hi = h ? hi_i : hi_r;
        uint8_t* pl = a0 + h * (OZP_HALF / 2) + off;
        constexpr int SL = OZP_HALF / 2 / OZ_NSL;  // 2 KB: one slice of this plane's half
        if constexpr (OZP_EPT == 4) {
          uint32_t l0[4], h0[4];
          transpose4(lo[0], lo[1], lo[2], lo[3], l0);
          transpose4(hi[0], hi[1], hi[2], hi[3], h0);
#pragma unroll
          for (int p = 0; p < 4; ++p) *reinterpret_cast<uint32_t*>(pl + p * SL) = l0[p];
#pragma unroll
          for (int p = 0; p < OZ_NSL - 4; ++p) *reinterpret_cast<uint32_t*>(pl + (4 + p) * SL) = h0[p];
        } else {
          uint32_t l0[4], l1[4], h0[4], h1[4];
          transpose4(lo[0], lo[1], lo[2], lo[3], l0);
          transpose4(lo[4], lo[5], lo[6], lo[7], l1);
          transpose4(hi[0], hi[1], hi[2], hi[3], h0);
          transpose4(hi[4], hi[5], hi[6], hi[7], h1);
#pragma unroll
          for (int p = 0; p < 4; ++p) *reinterpret_cast<uint2*>(pl + p * SL) = make_uint2(l0[p], l1[p]);
#pragma unroll
          for (int p = 0; p < OZ_NSL - 4; ++p) *reinterpret_cast<uint2*>(pl + (4 + p) * SL) = make_uint2(h0[p], h1[p]);
        }
      }
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      if (s == 0 && d > 0) drain(d - 1);
      asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
      __syncwarp();
      unsigned last = 0;
      if (lane == 0) {
        __threadfence_block();
        last = atomicAdd(&cnt[slot], 1u) == OZP_WARPS - 1;
        if (last) {
          cnt[slot] = 0;
          __threadfence_block();
          // the whole half is written: send it to the peer's slot
          const uint32_t src = sA + slot * OZ_ASTAGE + cr * OZP_HALF;
          if (!(OZ_EXP & 16)) bulk_s2peer(mapa_peer(src, peer), src, OZP_HALF, mapa_peer(fullA(slot), peer));
        }
      }
      if (__shfl_sync(0xffffffffu, last, 0)) {
        pend_slot = slot;
        pend_ph = ph;
        pend_s = s;
        pend_nst = nst;
      }
      __syncwarp();
    }
  }
  if (pend_slot >= 0) issue_stage(pend_slot, pend_ph, pend_s, pend_nst);
  __syncwarp();
  if (nchunks > 0) drain(nchunks - 1);
  if (KIND != KK_NUFFT && amp_hi >= amp_limit_hi<KIND>()) atomicOr(flag, 2);
  if (go < m_out && nchunks == 0) {
#pragma unroll
    for (int c = 0; c < DC; ++c)
      if (cb + c < it.ncols) Yb[yidx(c)] = 0.0;
  }
  // the peer's last multicast commits must have landed here before this CTA
  // exits: wait for the final phase of each slot's empty barrier
  if (g >= 1) mbar_wait(empty((g - 1) % OZ_NST), (uint32_t)((g - 1) / OZ_NST) & 1u);
  if (g >= 2) mbar_wait(empty((g - 2) % OZ_NST), (uint32_t)((g - 2) / OZ_NST) & 1u);
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  cluster_sync_all();
  if (warp == 0) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    if (cr == 0)
      asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(COLS0));
    else
      asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(COLS1));
  }
}

__global__ void oz_reduce_kernel(const double2* __restrict__ P, int64_t pstride, int nsplit, double2* Y, int64_t ldy,
                                 int64_t m, int64_t col0, int64_t ncols) {
  const int64_t total = m * ncols;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = t % m, c = t / m;
    const int64_t off = i + (col0 + c) * ldy;
    double2 s = P[off];
    for (int z = 1; z < nsplit; ++z) {
      const double2 v = P[z * pstride + off];
      s.x += v.x;
      s.y += v.y;
    }
    Y[off] = s;
  }
}

template <int KIND, int MODE, int NCB, bool PAIR>
bool run_oz(Ctx* c, Points outp, Points inp, double kappa, int64_t m_out, const double2* X, double2* Y, int64_t ldy,
            const MatvecSeg* segs, int nseg) {
  using Z = OzT<NCB, oz_kd(KIND), KIND == KK_PLATES>;
  std::vector<OzItem> items;
  std::vector<const MatvecSeg*> item_seg;
  int64_t max_rows = 0, max_col = 0, nstages = 0;
  for (int s = 0; s < nseg; ++s) {
    const MatvecSeg& g = segs[s];
    if (g.ncols <= 0) continue;
    if (g.rows <= 0) {
      BFLY_CUDA(cudaMemset2DAsync(Y + g.col0 * ldy, ldy * sizeof(double2), 0, m_out * sizeof(double2), g.ncols,
                                  c->stream));
      continue;
    }
    for (int tc = 0; tc < g.ncols; tc += NCB) {
      OzItem it{};
      it.row0 = g.row0;
      it.rows = g.rows;
      it.x_off = g.x_off + (int64_t)tc * g.ldx;
      it.ldx = g.ldx;
      it.ycol = g.col0 + tc;
      it.ncols = std::min(NCB, g.ncols - tc);
      it.bstage0 = nstages;
      nstages += ceil_div(g.rows, (int64_t)OZ_KS);
      items.push_back(it);
    }
    max_rows = std::max(max_rows, g.rows);
    max_col = std::max(max_col, g.col0 + (int64_t)g.ncols);
  }
  if (items.empty()) return true;
  if (items.size() > 65535) fail(PRECONDITION, "matvec: too many work items");
  const int64_t gx = ceil_div(m_out, (int64_t)OZ_BM);
  const int64_t base_ctas = gx * (int64_t)items.size();
  // split long segments so the grid covers every SM a few times (1 CTA / SM)
  const int64_t target = (int64_t)c->sm_count * 4;
  int nsplit = 1;
  if (base_ctas < target) nsplit = (int)std::min<int64_t>(ceil_div(target, base_ctas), ceil_div(max_rows, (int64_t)Z::KD));
  nsplit = std::max(1, std::min(nsplit, 64));
  const int64_t rows_per_split = ceil_div(ceil_div(max_rows, (int64_t)nsplit), (int64_t)Z::KD) * Z::KD;
  nsplit = (int)ceil_div(max_rows, rows_per_split);

  DBuf<OzItem> ditems(c, items.size());
  ditems.upload(items.data(), items.size());
  DBuf<int32_t> T(c, items.size() * OZ_MAXCB);
  DBuf<uint8_t> img(c, (size_t)(nstages * Z::BSTAGE));
  DBuf<int> local_flag;
  int* flag = c->oz_deferred ? c->oz_flag_dev() : nullptr;
  if (!flag) {
    local_flag.reset(c, 1);
    local_flag.zero();
    flag = local_flag.p;
  }
  double kflops = 0, kbytes = 0;
  for (const auto& it : items) {
    kflops += 8.0 * (double)m_out * (double)it.rows * (double)it.ncols;
    kbytes += 16.0 * ((double)it.rows + (double)m_out) * (double)it.ncols;
  }
  {
    KTimer timer(c, "oz_prep", 0.0, (double)nstages * Z::BSTAGE);
    oz_colscale_kernel<<<dim3(NCB, (unsigned)items.size()), 256, 0, c->stream>>>(X, ditems.p, T.p);
    BFLY_LAUNCH_CHECK("oz_colscale");
    const int64_t per_item = ceil_div(max_rows, (int64_t)OZ_KS) * 2 * NCB;
    oz_slice_kernel<NCB><<<dim3((unsigned)ceil_div(per_item, (int64_t)128), (unsigned)items.size()), 128, 0, c->stream>>>(
        X, ditems.p, T.p, img.p, flag);
    BFLY_LAUNCH_CHECK("oz_slice");
  }
  {
    static std::atomic<uint64_t> tab_ready{0};  // per device
    const uint64_t bit = uint64_t(1) << (c->device & 63);
    if (!(tab_ready.load() & bit)) {
      oz_table_kernel<<<keval::kTabN / 256, 256, 0, c->stream>>>();
      BFLY_LAUNCH_CHECK("oz_table");
      tab_ready.fetch_or(bit);
    }
  }
  static_assert(!PAIR || NCB == OZP_NCB || NCB == OZP_NCB48, "pair tile width");
  auto kern = PAIR ? matvec_oz_pair_kernel<KIND, MODE, NCB> : matvec_oz_kernel<KIND, MODE, NCB>;
  BFLY_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, Z::SM_TOTAL));
  dim3 grid((unsigned)(gx * (PAIR ? 2 : 1)), (unsigned)items.size(), (unsigned)nsplit);
  // partial output slices: split-K ranges, and the two diagonal halves of a pair
  const int nparts = nsplit * (PAIR ? 2 : 1);
  DBuf<double2> part;
  int64_t pstride = 0;
  double2* Yt = Y;
  if (nparts > 1) {
    pstride = ldy * max_col;
    part.reset(c, (size_t)(pstride * nparts));
    Yt = part.p;
  }
  // tensor work actually executed (int8 ops = 2 per MAC): per stage of 128
  // rows x 32 entries, 2 planes x (sum of MMA N) x 128 x 32 MACs
  double stages = 0;
  for (const auto& it : items)
    for (int z = 0; z < nsplit; ++z) {
      const int64_t k0 = (int64_t)z * rows_per_split, k1 = std::min(it.rows, k0 + rows_per_split);
      if (k1 > k0) stages += (double)ceil_div(k1 - k0, (int64_t)OZ_KS);
    }
  double nsum = 0;
  if (PAIR) {
    for (const OzSched& sch : {OzPairSched<0, NCB>::value, OzPairSched<1, NCB>::value})
      for (int i = 0; i < sch.n; ++i) nsum += (double)(((sch.code[i] >> 8) & 31) * Z::BN2);
  } else {
    constexpr OzSched sch = make_sched(Z::MAXB);
    for (int i = 0; i < sch.n; ++i) nsum += (double)(((sch.code[i] >> 8) & 31) * Z::BN2);
  }
  const double int8_ops = 2.0 * stages * (double)gx * nsum * OZ_BM * OZ_KS;
#ifdef OZ_TRACE
  {
    const char* om = std::getenv("BFLY_OZ_MODE");
    const int mode = om ? std::atoi(om) : 0;
    BFLY_CUDA(cudaMemcpyToSymbol(g_oz_mode, &mode, sizeof(int)));
  }
#endif
  {
    KTimer timer(c, "kernel_matvec", kflops, kbytes);
    KTimer timer8(c, "kernel_matvec.int8_ops", int8_ops, 0.0);
    BFLY_HOST_TRACE("K2 launch");
    if (PAIR) {
      cudaLaunchConfig_t cfg{};
      cfg.gridDim = grid;
      cfg.blockDim = dim3(PAIR ? OZP_THREADS : OZS_THREADS);
      cfg.dynamicSmemBytes = Z::SM_TOTAL;
      cfg.stream = c->stream;
      cudaLaunchAttribute attr[1];
      attr[0].id = cudaLaunchAttributeClusterDimension;
      attr[0].val.clusterDim.x = 2;
      attr[0].val.clusterDim.y = 1;
      attr[0].val.clusterDim.z = 1;
      cfg.attrs = attr;
      cfg.numAttrs = 1;
      BFLY_CUDA(cudaLaunchKernelEx(&cfg, kern, outp, inp, kappa, m_out, (const uint8_t*)img.p, (const int32_t*)T.p, Yt,
                                   ldy, (const OzItem*)ditems.p, rows_per_split, pstride, flag));
    } else {
      kern<<<grid, OZS_THREADS, Z::SM_TOTAL, c->stream>>>(outp, inp, kappa, m_out, img.p, T.p, Yt, ldy, ditems.p,
                                                      rows_per_split, pstride, flag);
    }
    BFLY_LAUNCH_CHECK("kernel_matvec_oz");
  }
  if (nparts > 1) {
    for (int s = 0; s < nseg; ++s) {
      const MatvecSeg& g = segs[s];
      if (g.ncols <= 0 || g.rows <= 0) continue;
      const int64_t total = m_out * g.ncols;
      const unsigned blocks = (unsigned)std::min<int64_t>(ceil_div(total, (int64_t)256), (int64_t)c->sm_count * 16);
      oz_reduce_kernel<<<blocks, 256, 0, c->stream>>>(part.p, pstride, nparts, Y, ldy, m_out, g.col0, g.ncols);
      BFLY_LAUNCH_CHECK("oz_reduce");
    }
  }
#ifdef OZ_TRACE
  {
    unsigned long long tr[8];
    const char* om = std::getenv("BFLY_OZ_MODE");
    const int mode = om ? std::atoi(om) : 0;
    (void)mode;
    c->sync();
    BFLY_CUDA(cudaMemcpyFromSymbol(tr, g_oz_trace, sizeof(tr)));
    const double ctas = (double)gx * items.size() * nsplit;
    fprintf(stderr,
            "[oz] ctas %.0f per-CTA cycles: total %.0f | per warp: eval %.0f write %.0f wait-empty %.0f accF %.0f "
            "setup %.0f | issuer: issue %.0f ticket %.0f (per CTA)\n",
            ctas, tr[5] / ctas, tr[0] / ctas / OZ_EWARPS, tr[1] / ctas / OZ_EWARPS, tr[3] / ctas / OZ_EWARPS,
            tr[4] / ctas / OZ_EWARPS, tr[6] / ctas / OZ_EWARPS, tr[2] / ctas, tr[7] / ctas);
    unsigned long long z[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    BFLY_CUDA(cudaMemcpyToSymbol(g_oz_trace, z, sizeof(z)));
  }
#endif
  if (std::getenv("BFLY_OZ_TEST_OVERFLOW"))  // test hook: exercise the FP64 recompute path
    BFLY_CUDA(cudaMemsetAsync(flag, 0xFF, sizeof(int), c->stream));
  if (c->oz_deferred) return true;  // checked once per factorization (Ctx::take_oz_overflow)
  int hflag = 0;
  local_flag.download(&hflag, 1);
  c->sync();
  return hflag == 0;
}

bool oz_pair_enabled() {
  const char* e = std::getenv("BFLY_OZ_PAIR");
  return !(e && std::string(e) == "0");
}

template <int KIND, int MODE>
bool run_oz_width(Ctx* c, Points outp, Points inp, double kappa, int64_t m_out, const double2* X, double2* Y,
                  int64_t ldy, const MatvecSeg* segs, int nseg) {
  // tile width = the widest column tile of the launch: narrow probe blocks
  // (leaf rounds) do proportionally less tensor work; 33..40 columns run on
  // CTA pairs (one evaluation for all of them), wider blocks in 32-column tiles
  int w = 0;
  for (int s = 0; s < nseg; ++s) w = std::max(w, std::min(segs[s].ncols, OZ_MAXCB));
  if (w <= 8) return run_oz<KIND, MODE, 8, false>(c, outp, inp, kappa, m_out, X, Y, ldy, segs, nseg);
  if (w <= 16) return run_oz<KIND, MODE, 16, false>(c, outp, inp, kappa, m_out, X, Y, ldy, segs, nseg);
  if (w <= 24) return run_oz<KIND, MODE, 24, false>(c, outp, inp, kappa, m_out, X, Y, ldy, segs, nseg);
  if (w > OZ_MAXCB1 && w <= OZP_NCB && oz_pair_enabled())
    return run_oz<KIND, MODE, OZP_NCB, true>(c, outp, inp, kappa, m_out, X, Y, ldy, segs, nseg);
  if constexpr (KIND == KK_PLATES)
    if (w > OZP_NCB && w <= OZP_NCB48 && oz_pair_enabled())
      return run_oz<KIND, MODE, OZP_NCB48, true>(c, outp, inp, kappa, m_out, X, Y, ldy, segs, nseg);
  return run_oz<KIND, MODE, 32, false>(c, outp, inp, kappa, m_out, X, Y, ldy, segs, nseg);
}

template <int KIND>
bool dispatch_oz_mode(Ctx* c, int mode, Points outp, Points inp, double kappa, int64_t m_out, const double2* X,
                      double2* Y, int64_t ldy, const MatvecSeg* segs, int nseg) {
  if (mode == OP_N) return run_oz_width<KIND, OP_N>(c, outp, inp, kappa, m_out, X, Y, ldy, segs, nseg);
  if (mode == OP_T) return run_oz_width<KIND, OP_T>(c, outp, inp, kappa, m_out, X, Y, ldy, segs, nseg);
  return run_oz_width<KIND, OP_H>(c, outp, inp, kappa, m_out, X, Y, ldy, segs, nseg);
}

}  // namespace

int kernel_matvec_pass_cols() { return matvec_oz_enabled() && oz_pair_enabled() ? OZP_NCB : OZ_MAXCB1; }

bool matvec_oz_enabled() {
  const char* e = std::getenv("BFLY_MATVEC");
  return !(e && std::string(e) == "fp64");
}

bool launch_kernel_matvec_oz(Ctx* c, int kind, int mode, Points outp, Points inp, double kappa, int64_t m_out,
                             const double2* X, double2* Y, int64_t ldy, const MatvecSeg* segs, int nseg) {
  if (m_out <= 0 || nseg <= 0) return true;
  if (kind == KK_NUFFT) return dispatch_oz_mode<KK_NUFFT>(c, mode, outp, inp, kappa, m_out, X, Y, ldy, segs, nseg);
  if (kind == KK_PLATES) return dispatch_oz_mode<KK_PLATES>(c, mode, outp, inp, kappa, m_out, X, Y, ldy, segs, nseg);
  if (kind == KK_CIRCLE) return dispatch_oz_mode<KK_CIRCLE>(c, mode, outp, inp, kappa, m_out, X, Y, ldy, segs, nseg);
  fail(PRECONDITION, "kernel_matvec: unknown kernel kind");
  return false;
}

}  // namespace bfly
