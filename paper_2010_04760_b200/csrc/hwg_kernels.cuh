// Fused RHS + SSP-RK stage kernels for the first-order (rho, theta) Teukolsky
// system (B200 / sm_100a).
//
// One launch = one RK stage over the whole (slab) grid:
//   u_out = epilogue(u_n, ..., u_k, F(u_k))
// where F is EvolutionRhs::operator() (proj/src/evolve.cpp:181-187): ghost
// fill (evolve.cpp:40-71) + radial WENO5/WENO3/FD6 derivatives (phase 1,
// evolve.cpp:88-122) + theta operator on Psi (phase 2, :125-136) + pointwise
// assembly with the 9 coefficient planes and KO8 (phase 3, :139-178), and the
// epilogue is one of the stage updates of ssprk33_step / ssprk104_step
// (proj/include/hweno/timestep.hpp:54-109).  Nothing touches HBM between the
// phases: one stage reads u_k (+ u_n, ...) and the coefficients once and
// writes u_out once.
//
// Device layout: theta fastest, blocked by 32-column chunks.
//   state register: block (row r, chunk c) = 64 double2 = [Psi(32) | pi(32)],
//     Psi = (Psi_R, Psi_I), pi = (pi_R, pi_I); rows r in [-kHalo, n + kHalo),
//     block index (r + kHalo) * nchunks + c, so one row is contiguous.
//   coefficients: block (row j, chunk c) = 2304 B = [(b,lam) | (w_re,w_im) |
//     (bt_re,bt_im) | (c_re,c_im) | ath], 32 columns each.
// A warp's whole per-row input is therefore 3 contiguous blocks (coefficients,
// u_n, the next stencil row), moved by 3 bulk copies.
//
// Work decomposition: a warp owns one chunk and a contiguous range of rows;
// each lane owns one theta column and marches along rho with a register
// window of the stencil rows, so every state value is read from HBM once
// (plus the halo rows of each range).  Theta neighbours come from a per-warp
// shared-memory row (parity-reflected at the poles, evolve.cpp:59-70); the
// four lanes at the chunk edges fetch the neighbouring chunks' columns one row
// ahead.  Radial
// ghosts at the physical ends are synthesised in registers with the
// reference's cubic recurrence (evolve.cpp:45-57); slab ends read halo rows.
//
// Arithmetic: compiled with -fmad=false; every fused multiply-add below is an
// explicit fma(), so an interface's value does not depend on where it is
// computed (slab boundaries reproduce the single-GPU result bitwise).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>  // device printf of the HWG_DEBUG bounds checks

#ifndef HWG_MINB
// resident blocks per SM: 3 (12 warps at up to 168 registers, room for the
// 2-row unrolled loop) measured 2-4 % faster than 4 (16 warps at 128)
#define HWG_MINB 3
#endif
#ifndef HWG_RING
#define HWG_RING 2  // bulk-copy ring depth per warp (measured: 2 beats 3 and 4 by 1-2 %)
#endif

namespace hwg {

constexpr int kHalo = 4;          // halo rows per side (KO8 needs 4)
constexpr int kWarpsPerBlock = 4;
constexpr unsigned kFull = 0xffffffffu;
constexpr int kStateBlk = 64;     // double2 per (row, chunk) state block
constexpr int kCoefBlk = 144;     // double2 per (row, chunk) coefficient block
constexpr int kCoefAth = 128;     // ath offset (double2 units) in a coefficient block

enum SchemeId { WENO5 = 0, WENO3 = 1, FD6KO = 2 };
// F64: fp64 weights.  MIXED: fp32 weights (the paper's mode).  LIN: eps = inf,
// frozen linear weights (spatial.hpp:15-18, 33-38).
enum ModeId { F64 = 0, MIXED = 1, LIN = 2 };
enum EpiId {
  EPI_RHS = 0,       // o = f                                       (EvolutionRhs)
  EPI_AXPY = 1,      // o = x + g f                                 (rk33 stage 1, rk104 i)
  EPI_RK3 = 2,       // o = a A + b (x + g f)                       (rk33 stage 2)
  EPI_RK3C = 3,      // rk33 stage 3 + admissibility scan
  EPI_RK104_5 = 4,   // o = a A + b x + g f ; F4 = f                (rk104 stage 5)
  EPI_RK104_10 = 5   // o = a A + b B + c x + g (d G + e f) + scan  (rk104 stage 10)
};

// Slab neighbours over peer memory (multi-GPU radial slabs).
// The stage kernel itself stores its first / last h output rows into the
// neighbours' halo rows of the same register and bumps their arrival counter;
// the next stage's boundary warps wait on their own counters before reading
// halo rows.  Counters are monotonic: after e stages every neighbour has
// signalled e * nchunks times (one per chunk), so a boundary warp at epoch e
// waits for >= e * nchunks.
struct PeerArgs {
  double2* o_lo;                   // lower neighbour's output register at its row n_lo
  double2* o_hi;                   // upper neighbour's output register at its row -h
  unsigned long long* sig_lo;      // lower neighbour's "from upper" counter
  unsigned long long* sig_hi;      // upper neighbour's "from lower" counter
  unsigned long long* wait;        // own counters: [0] from lower, [1] from upper (flag + 6)
  unsigned long long* epoch;       // own epoch (flag + 5)
  long long timeout_ns;            // bounded spin: flag[0] |= 2 on expiry
  int h;                           // halo rows pushed per side
  int on_lo, on_hi;                // neighbour present
};

struct StageArgs {
  int n, nt, nchunks;
  long long rs, crs;               // double2 per state / coefficient row (row pitch)
  int phys_lo, phys_hi;            // slab holds the excision / scri end
  int nranges;
  int negpar;                      // theta parity (-1)^(m+s) == -1
  long long step;                  // blowup_step recorded if the scan fails; < 0: use flag[2]
  int bump;                        // stage 0 in counter mode: flag[2] += 1 (graph replay)
  double eps4;                     // fp64 weights: 4 eps (scaled indicators)
  double eps;                      // fp64 weno3
  float epsf;                      // fp32 weights: eps demoted
  double ko;                       // KO8: sigma / (256 drho)
  double ca, cb, cc, cg, cd, ce;   // epilogue coefficients
  // state registers at row 0 (halo rows at negative offsets), blocked layout
  const double2* x;                // stencil input u_k
  const double2* ua;               // u_n
  const double2* ub;               // u^(4)
  const double2* ug;               // F(u^(4))
  double2* o;                      // output
  double2* f;                      // F store (rk104 stage 5)
  const double2* coef;             // coefficient blocks, rows [0, n)
  const double* cot;               // cot(theta_k), padded to nchunks*32
  unsigned long long* flag;        // [0] blown, [1] blowup step, [2] step counter, [3] pending
  // end-of-launch ticket (flag + 4): the last warp publishes the pending
  // blow-up bit (so every block of a launch sees the same frozen state) and
  // advances the peer epoch.  Null for launches that need neither.
  unsigned long long* tick;
  PeerArgs px;                     // fused halo push to the neighbour slabs (NVLink P2P)
  int pdl;                         // launched with programmatic stream serialisation
  // row window of this launch: [row_lo, row_hi) of the slab (the whole slab,
  // or one part of a stage split around an overlapped halo exchange)
  int row_lo, row_hi;
  int defer;                       // not the stage's last part: blow-up bit stays pending
};

__device__ __forceinline__ double2 ld2(const double2* p) { return __ldg(p); }

// Debug builds (-DHWG_DEBUG, tools/build_variant.sh dbg -DHWG_DEBUG): every
// global address the stage kernel forms is checked against the extent of the
// array it points into, trapping on a violation (compute-sanitizer is not
// available on the GPU pool; the GPU test suite runs against this build).
#ifdef HWG_DEBUG
#define HWG_CHK(cond)                                                                    \
  do {                                                                                   \
    if (!(cond)) {                                                                       \
      printf("hwg bounds check failed: %s (line %d, block %d, thread %d)\n", #cond,      \
             __LINE__, blockIdx.x, threadIdx.x);                                         \
      asm volatile("trap;");                                                             \
    }                                                                                    \
  } while (0)
#else
#define HWG_CHK(cond) \
  do {                \
  } while (0)
#endif
// p .. p + len (double2) inside a state register given by its row-0 pointer
__device__ __forceinline__ bool in_reg(const double2* p, const double2* row0, ptrdiff_t rs, int n,
                                       int len) {
  return p >= row0 - kHalo * rs && p + len <= row0 + (ptrdiff_t)(n + kHalo) * rs;
}
__device__ __forceinline__ double2 neg2(double2 v) { return make_double2(-v.x, -v.y); }

// reference cubic continuation p[-t] = 4p[-t+1] - 6p[-t+2] + 4p[-t+3] - p[-t+4]
// (evolve.cpp:48-50), same evaluation order
__device__ __forceinline__ double cubic1(double a, double b, double c, double d) {
  return 4.0 * a - 6.0 * b + 4.0 * c - d;
}
__device__ __forceinline__ double2 cubic(double2 a, double2 b, double2 c, double2 d) {
  return make_double2(cubic1(a.x, b.x, c.x, d.x), cubic1(a.y, b.y, c.y, d.y));
}

// pi value of row r of one column (col = this lane's pi at row 0, rstride =
// double2 per row); rows < 0 of the slab holding the excision end are the
// reference's cubic ghosts.  Rare path: the orientation switch of a pi row.
static __device__ __noinline__ double2 row_or_ghost(const double2* col, int r, ptrdiff_t rstride,
                                             int phys_lo) {
  if (r >= 0 || !phys_lo) return __ldcg(col + r * rstride);  // may be a peer-written halo row
  double2 g[8];
  for (int m = 0; m < 4; ++m) g[4 + m] = __ldg(col + m * rstride);
  for (int t = 1; t <= -r; ++t)
    g[4 - t] = cubic(g[4 - t + 1], g[4 - t + 2], g[4 - t + 3], g[4 - t + 4]);
  return g[4 + r];
}

// ---------------------------------------------------------------------------
// Reciprocals without IEEE special-case branches.  The arguments below are
// sums of positive weights (never 0, inf or subnormal on admissible states);
// a NaN state still propagates NaN.
__device__ __forceinline__ float frcp(float x) {
  float r;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}
__device__ __forceinline__ double drcp(double x) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));  // MUFU.RCP64H seed (~2^-20)
  double e = fma(-x, r, 1.0);
  r = fma(r, e, r);                                       // ~2^-40
  e = fma(-x, r, 1.0);
  return fma(r, e, r);                                    // ~1 ulp
}

// ---------------------------------------------------------------------------
// WENO5-JS interface values (spatial.hpp:29-92) of both components of an
// oriented window f0..f4 (double2 = real, imaginary), returned WITHOUT the
// 1/6 factor (folded with 1/drho into the coefficient planes b, lam, w).
//
// F64: alpha_k = d_k/(eps + IS_k)^2 normalised.  With the indicators scaled
// by 4 (IS' = 13/3 t^2 + s^2, eps' = 4 eps) the weights are
// w_k = d_k prod_{i!=k} e_i^2 / sum(...), so one reciprocal replaces the
// reference's five divisions (weights and renormalisation, spatial.hpp:58-90).
__device__ __forceinline__ double weno5_f64(double f0, double f1, double f2, double f3,
                                            double f4, double eps4) {
  const double c = 13.0 / 3.0;
  double t0 = fma(-2.0, f1, f0) + f2;
  double s0 = fma(3.0, f2, fma(-4.0, f1, f0));
  double t1 = fma(-2.0, f2, f1) + f3;
  double s1 = f1 - f3;
  double t2 = fma(-2.0, f3, f2) + f4;
  double s2 = fma(3.0, f2, fma(-4.0, f3, f4));
  double e0 = fma(s0, s0, fma(c * t0, t0, eps4));
  double e1 = fma(s1, s1, fma(c * t1, t1, eps4));
  double e2 = fma(s2, s2, fma(c * t2, t2, eps4));
  double q0 = e0 * e0, q1 = e1 * e1, q2 = e2 * e2;
  double n0 = q1 * q2;
  double n1 = 6.0 * (q0 * q2);
  double n2 = 3.0 * (q0 * q1);
  double c0 = fma(11.0, f2, fma(-7.0, f1, 2.0 * f0));
  double c1 = fma(2.0, f3, fma(5.0, f2, -f1));
  double c2 = fma(5.0, f3, fma(2.0, f2, -f4));
  double num = fma(n2, c2, fma(n1, c1, n0 * c0));
  return num * drcp((n0 + n1) + n2);
}

// linear weights (1/10, 6/10, 3/10): the eps = inf reconstruction
__device__ __forceinline__ double weno5_lin(double f0, double f1, double f2, double f3, double f4) {
  double c0 = fma(11.0, f2, fma(-7.0, f1, 2.0 * f0));
  double c1 = fma(2.0, f3, fma(5.0, f2, -f1));
  double c2 = fma(5.0, f3, fma(2.0, f2, -f4));
  return fma(0.3, c2, fma(0.6, c1, 0.1 * c0));
}

__device__ __forceinline__ float2 f2(float x) { return make_float2(x, x); }

// 1 / s for a sum s = 1 + d of promoted fp32 weights that were normalised in
// fp32 (|d| <= a few fp32 ulps, ~1e-6): 1 - d + d^2 is exact to ~d^3 < 1e-18,
// below fp64 rounding, in two dependent FP64 ops instead of a reciprocal
// (the reference's renormalisation in work precision, spatial.hpp:84-90).
// s - 1 is exact (Sterbenz); a NaN sum stays NaN.
__device__ __forceinline__ double renorm_inv(double s) {
  const double d = s - 1.0;
  return fma(d, d, 1.0 - d);
}
__device__ __forceinline__ float2 dem2(double2 v) { return make_float2((float)v.x, (float)v.y); }

// MIXED (the paper's mode): window demoted to fp32, smoothness indicators
// and nonlinear weights in fp32 (spatial.hpp:29-65 with TW = float), promoted
// and renormalised in fp64 work precision (:84-90), fp64 candidate stencils.
// The real and imaginary components share the schedule, so the fp32 work runs
// on Blackwell's packed FP32x2 pipe (FFMA2 / FMUL2 / FADD2).
__device__ __forceinline__ double2 weno5_mixed2(double2 f0, double2 f1, double2 f2_, double2 f3,
                                                double2 f4, float eps) {
  const float2 g0 = dem2(f0), g1 = dem2(f1), g2 = dem2(f2_), g3 = dem2(f3), g4 = dem2(f4);
  // indicators scaled by 4 (E = 4 (eps + IS) = 13/3 t^2 + s^2 + 4 eps): the
  // weights are invariant under the common factor 16 of the alphas
  const float2 c133 = f2(13.0f / 3.0f), ep = f2(4.0f * eps);
  float2 t = __fadd2_rn(__ffma2_rn(f2(-2.0f), g1, g0), g2);
  float2 s = __ffma2_rn(f2(3.0f), g2, __ffma2_rn(f2(-4.0f), g1, g0));
  float2 e0 = __ffma2_rn(__fmul2_rn(c133, t), t, __ffma2_rn(s, s, ep));
  t = __fadd2_rn(__ffma2_rn(f2(-2.0f), g2, g1), g3);
  s = __ffma2_rn(f2(-1.0f), g3, g1);
  float2 e1 = __ffma2_rn(__fmul2_rn(c133, t), t, __ffma2_rn(s, s, ep));
  t = __fadd2_rn(__ffma2_rn(f2(-2.0f), g3, g2), g4);
  s = __ffma2_rn(f2(3.0f), g2, __ffma2_rn(f2(-4.0f), g3, g4));
  float2 e2 = __ffma2_rn(__fmul2_rn(c133, t), t, __ffma2_rn(s, s, ep));
  const float2 q0 = __fmul2_rn(e0, e0), q1 = __fmul2_rn(e1, e1), q2 = __fmul2_rn(e2, e2);
  const float2 a0 = __fmul2_rn(f2(0.1f), make_float2(frcp(q0.x), frcp(q0.y)));
  const float2 a1 = __fmul2_rn(f2(0.6f), make_float2(frcp(q1.x), frcp(q1.y)));
  const float2 a2 = __fmul2_rn(f2(0.3f), make_float2(frcp(q2.x), frcp(q2.y)));
  const float2 sm = __fadd2_rn(__fadd2_rn(a0, a1), a2);
  const float2 inv = make_float2(frcp(sm.x), frcp(sm.y));
  const float2 w0 = __fmul2_rn(a0, inv), w1 = __fmul2_rn(a1, inv), w2 = __fmul2_rn(a2, inv);
  double2 out;
  {
    const double W0 = w0.x, W1 = w1.x, W2 = w2.x;
    double c0 = fma(11.0, f2_.x, fma(-7.0, f1.x, 2.0 * f0.x));
    double c1 = fma(2.0, f3.x, fma(5.0, f2_.x, -f1.x));
    double c2 = fma(5.0, f3.x, fma(2.0, f2_.x, -f4.x));
    out.x = fma(W2, c2, fma(W1, c1, W0 * c0)) * renorm_inv((W0 + W1) + W2);
  }
  {
    const double W0 = w0.y, W1 = w1.y, W2 = w2.y;
    double c0 = fma(11.0, f2_.y, fma(-7.0, f1.y, 2.0 * f0.y));
    double c1 = fma(2.0, f3.y, fma(5.0, f2_.y, -f1.y));
    double c2 = fma(5.0, f3.y, fma(2.0, f2_.y, -f4.y));
    out.y = fma(W2, c2, fma(W1, c1, W0 * c0)) * renorm_inv((W0 + W1) + W2);
  }
  return out;
}

// WENO3 (spatial.hpp:94-130), without the 1/2 (folded into b, lam, w)
__device__ __forceinline__ double weno3_f64(double f0, double f1, double f2, double eps) {
  double d0 = f1 - f0, d1 = f2 - f1;
  double e0 = fma(d0, d0, eps), e1 = fma(d1, d1, eps);
  double n0 = e1 * e1, n1 = 2.0 * (e0 * e0);
  return fma(n1, f1 + f2, n0 * fma(3.0, f1, -f0)) * drcp(n0 + n1);
}
__device__ __forceinline__ double weno3_lin(double f0, double f1, double f2) {
  return fma(2.0 / 3.0, f1 + f2, (1.0 / 3.0) * fma(3.0, f1, -f0));
}
__device__ __forceinline__ double2 weno3_mixed2(double2 f0, double2 f1, double2 f2_, float eps) {
  const float2 g0 = dem2(f0), g1 = dem2(f1), g2 = dem2(f2_), ep = f2(eps);
  const float2 d0 = __ffma2_rn(f2(-1.0f), g0, g1);
  const float2 d1 = __ffma2_rn(f2(-1.0f), g1, g2);
  const float2 e0 = __ffma2_rn(d0, d0, ep), e1 = __ffma2_rn(d1, d1, ep);
  const float2 q0 = __fmul2_rn(e0, e0), q1 = __fmul2_rn(e1, e1);
  const float2 a0 = __fmul2_rn(f2(1.0f / 3.0f), make_float2(frcp(q0.x), frcp(q0.y)));
  const float2 a1 = __fmul2_rn(f2(2.0f / 3.0f), make_float2(frcp(q1.x), frcp(q1.y)));
  const float2 sm = __fadd2_rn(a0, a1);
  const float2 inv = make_float2(frcp(sm.x), frcp(sm.y));
  const float2 x0 = __fmul2_rn(a0, inv), x1 = __fmul2_rn(a1, inv);
  double2 out;
  out.x = fma((double)x1.x, f1.x + f2_.x, (double)x0.x * fma(3.0, f1.x, -f0.x)) *
          renorm_inv((double)x0.x + (double)x1.x);
  out.y = fma((double)x1.y, f1.y + f2_.y, (double)x0.y * fma(3.0, f1.y, -f0.y)) *
          renorm_inv((double)x0.y + (double)x1.y);
  return out;
}

template <int SCH, int MODE>
__device__ __forceinline__ double2 weno2(const double2 f0, const double2 f1, const double2 f2_,
                                         const double2 f3, const double2 f4, const StageArgs& a) {
  if (SCH == WENO5) {
    if (MODE == MIXED) return weno5_mixed2(f0, f1, f2_, f3, f4, a.epsf);
    if (MODE == LIN)
      return make_double2(weno5_lin(f0.x, f1.x, f2_.x, f3.x, f4.x),
                          weno5_lin(f0.y, f1.y, f2_.y, f3.y, f4.y));
    return make_double2(weno5_f64(f0.x, f1.x, f2_.x, f3.x, f4.x, a.eps4),
                        weno5_f64(f0.y, f1.y, f2_.y, f3.y, f4.y, a.eps4));
  }
  // WENO3 uses f0..f2 only
  if (MODE == MIXED) return weno3_mixed2(f0, f1, f2_, a.epsf);
  if (MODE == LIN)
    return make_double2(weno3_lin(f0.x, f1.x, f2_.x), weno3_lin(f0.y, f1.y, f2_.y));
  return make_double2(weno3_f64(f0.x, f1.x, f2_.x, a.eps), weno3_f64(f0.y, f1.y, f2_.y, a.eps));
}

// interface j + 1/2 + shift of both components from a double2 window whose
// row j sits at index C; minus = right-biased mirror (spatial.hpp:144-151)
template <int SCH, int MODE, int C>
__device__ __forceinline__ double2 iface2_at(const double2* w, bool minus, int shift,
                                             const StageArgs& a) {
  const int c = C + shift;
  if (SCH == WENO5)
    return minus ? weno2<SCH, MODE>(w[c + 3], w[c + 2], w[c + 1], w[c], w[c - 1], a)
                 : weno2<SCH, MODE>(w[c - 2], w[c - 1], w[c], w[c + 1], w[c + 2], a);
  return minus ? weno2<SCH, MODE>(w[c + 2], w[c + 1], w[c], w[c], w[c], a)
               : weno2<SCH, MODE>(w[c - 1], w[c], w[c + 1], w[c], w[c], a);
}

// ---------------------------------------------------------------------------
template <int SCH>
struct Win {
  // register windows, rows j - L .. j + R (L + R >= 4 so the cubic scri
  // continuation always has its four predecessors in registers)
  static constexpr int SL = (SCH == FD6KO) ? 4 : (SCH == WENO5 ? 1 : 2);  // Psi
  static constexpr int PL = (SCH == FD6KO) ? 4 : 2;                       // pi
  static constexpr int R = (SCH == FD6KO) ? 4 : (SCH == WENO5 ? 3 : 2);
  static constexpr int SW = SL + R + 1, PW = PL + R + 1;
  // rows needed at initialisation (fresh F(jb - 1/2) in either orientation)
  static constexpr int IL = (SCH == FD6KO) ? 4 : (SCH == WENO5 ? 3 : 2);
  static constexpr int IW = IL + R + 1;
  static constexpr int IA = (IL + 4 > IW) ? IL + 4 : IW;  // + 4 rows for the cubic
};

// parity reflection of a theta column across the poles (evolve.cpp:59-70)
__device__ __forceinline__ int reflect_col(int c, int nt, bool& flip, int negpar) {
  flip = false;
  if (c < 0) { c = -1 - c; flip = negpar; }
  else if (c >= nt) { c = 2 * nt - 1 - c; flip = negpar; }
  if (c < 0 || c >= nt) { c = 0; flip = false; }  // only for lanes far outside tiny grids
  return c;
}
// offset (double2) of the Psi value of column col inside a state row
__device__ __forceinline__ int psi_off(int col) { return (col >> 5) * kStateBlk + (col & 31); }

// ---------------------------------------------------------------------------
// Bulk-copy (TMA engine) row ring.  Each warp owns S slots of shared memory;
// slot s holds, for one iteration j: the coefficient block of row j, the
// state blocks of row j that the epilogue needs (u_n, u^(4), F(u^(4))) and
// the stencil-input block of row j + 1 + R that enters the register window
// at the end of the iteration.  Lane 0 issues the row's cp.async.bulk copies
// S iterations ahead; an mbarrier per slot completes on the byte count.  The
// lanes read their own column from shared memory, so the prefetch costs no
// registers and no per-lane memory instructions.
template <int EPI>
struct Slot {
  static constexpr int COEF = 0;                       // 2304 B
  static constexpr int XN = kCoefBlk * 16;             // next stencil row block, 1024 B
  static constexpr int A = XN + kStateBlk * 16;        // u_n
  static constexpr bool HAS_A = EPI >= EPI_RK3;
  static constexpr bool HAS_BG = EPI == EPI_RK104_10;
  static constexpr int B = A + (HAS_A ? kStateBlk * 16 : 0);
  static constexpr int G = B + kStateBlk * 16;
  static constexpr int BYTES = B + (HAS_BG ? 2 * kStateBlk * 16 : 0);
  static constexpr int S = HAS_BG ? 2 : HWG_RING;      // ring depth
};

// shared memory per block: the warps' rings, their mbarriers, then (16-byte
// aligned) per warp the theta-extended Psi row (36 double2) of the theta operator
template <int EPI>
__host__ __device__ constexpr size_t stage_theta_offset(int wpb) {
  return ((size_t)wpb * Slot<EPI>::S * (Slot<EPI>::BYTES + 8) + 15) & ~(size_t)15;
}
template <int EPI>
constexpr size_t stage_smem_bytes(int wpb = kWarpsPerBlock) {
  return stage_theta_offset<EPI>(wpb) + (size_t)wpb * 36 * 16;
}

// one lane of the (converged) warp, known to the compiler as a single lane
__device__ __forceinline__ bool elect_one() {
  uint32_t pred = 0;
  asm volatile(
      "{\n\t.reg .pred P;\n\telect.sync _|P, 0xffffffff;\n\tselp.u32 %0, 1, 0, P;\n}"
      : "=r"(pred));
  return pred != 0;
}
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes)
               : "memory");
}
// expected bytes without arriving (the arrival comes with the later copies)
__device__ __forceinline__ void mbar_expect_tx_only(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.expect_tx.relaxed.cta.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint32_t bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}
// programmatic dependent launch: let the next stage's grid launch now; wait
// for the previous stage's grid (and its memory) before touching its outputs
__device__ __forceinline__ void pdl_trigger() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred P1;\n"
      "WAIT_LOOP:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
      "@!P1 bra WAIT_LOOP;\n}" ::"r"(bar),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void* src, uint32_t bytes,
                                         uint32_t bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
      "l"(src), "r"(bytes), "r"(bar)
      : "memory");
}

__device__ __forceinline__ void peer_signal(unsigned long long* ctr, unsigned long long v) {
  asm volatile("red.release.sys.global.add.u64 [%0], %1;" ::"l"(ctr), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_acquire_sys(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ unsigned long long globaltimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
// bounded spin until *ctr >= want; false on timeout.  A wait that had to
// spin (the neighbour's rows were not there yet) is counted in *spun.
static __device__ __noinline__ bool peer_wait(const unsigned long long* ctr, unsigned long long want,
                                       long long timeout_ns, unsigned long long* spun) {
  if (ld_acquire_sys(ctr) >= want) return true;
  atomicAdd(spun, 1ull);
  const unsigned long long t0 = globaltimer();
  while (ld_acquire_sys(ctr) < want) {
    __nanosleep(200);
    if ((long long)(globaltimer() - t0) > timeout_ns) return false;
  }
  return true;
}

// boundary warps: wait for the neighbours' halo rows of this stage
static __device__ __noinline__ void peer_wait_halos(unsigned long long* wait,
                                                    const unsigned long long* epoch,
                                                    unsigned long long* flag, int nchunks,
                                                    long long timeout_ns, bool lo, bool hi) {
  if ((threadIdx.x & 31) == 0) {
    const unsigned long long want = *(volatile const unsigned long long*)epoch *
                                    (unsigned long long)nchunks;
    bool ok = true;
    if (lo) ok &= peer_wait(wait, want, timeout_ns, flag + 8);
    if (hi) ok &= peer_wait(wait + 1, want, timeout_ns, flag + 8);
    if (!ok) atomicOr(flag, 2ull);
    // the halo rows also arrive through the bulk-copy (async) proxy
    asm volatile("fence.proxy.async.global;" ::: "memory");
  }
  __syncwarp();
}

// push the boundary output rows this warp just wrote (its own stores, read
// back by the same lanes) into the neighbours' halo rows over NVLink, then
// signal their arrival counters
static __device__ __noinline__ void peer_push_halos(const double2* o, double2* o_lo,
                                                    double2* o_hi, unsigned long long* sig_lo,
                                                    unsigned long long* sig_hi, ptrdiff_t rs,
                                                    int n, int nt, int h, int chunk, bool lo,
                                                    bool hi) {
  const int lane = threadIdx.x & 31;
  const ptrdiff_t c = chunk * kStateBlk + lane;
  const double2* ob = o + c;
  if ((chunk << 5) + lane < nt) {
    for (int r = 0; lo && r < h; ++r) {
      o_lo[r * rs + c] = ob[r * rs];
      o_lo[r * rs + c + 32] = ob[r * rs + 32];
    }
    for (int r = 0; hi && r < h; ++r) {
      o_hi[r * rs + c] = ob[(n - h + r) * rs];
      o_hi[r * rs + c + 32] = ob[(n - h + r) * rs + 32];
    }
  }
  __threadfence_system();
  __syncwarp();
  if (lane == 0) {
    if (lo) peer_signal(sig_lo, 1ull);
    if (hi) peer_signal(sig_hi, 1ull);
  }
}

// every warp of a launch (nw warps) takes a ticket; the last one publishes
// the pending blow-up bit and advances the peer epoch
static __device__ __noinline__ void launch_ticket(unsigned long long* tick,
                                                  unsigned long long* flag,
                                                  unsigned long long* epoch,
                                                  unsigned long long nw) {
  __syncwarp();
  if ((threadIdx.x & 31) == 0) {
    __threadfence();
    if (atomicAdd(tick, 1ull) == nw - 1) {
      __threadfence();
      if (atomicExch(flag + 3, 0ull) != 0ull) atomicOr(flag, 1ull);
      if (epoch != nullptr) *epoch += 1ull;
      *tick = 0ull;
    }
  }
}

template <int SCH, int MODE, int EPI, class WaitIn>
__device__ __forceinline__ bool stage_body(const StageArgs& a, unsigned char* ring, uint32_t bar0,
                                           double2* trow, WaitIn&& wait_in, int bid);

// shared memory of one warp for a whole-launch stage: its ring, its ring's
// mbarriers, its theta row (stage_smem_bytes)
template <int EPI>
__device__ __forceinline__ void stage_layout(unsigned char*& ring, uint32_t& bar0,
                                             double2*& trow) {
  extern __shared__ __align__(128) unsigned char smem[];
  constexpr int S = Slot<EPI>::S, SB = Slot<EPI>::BYTES;
  const int wib = threadIdx.x >> 5, wpb = blockDim.x >> 5;
  ring = smem + (size_t)wib * S * SB;
  bar0 = smem_u32(smem + (size_t)wpb * S * SB) + wib * S * 8;
  trow = reinterpret_cast<double2*>(smem + stage_theta_offset<EPI>(wpb)) + wib * 36;
}

template <int SCH, int MODE, int EPI>
__global__ void __launch_bounds__(kWarpsPerBlock * 32, HWG_MINB)
stage_kernel(const StageArgs a) {
  unsigned char* ring;
  uint32_t bar0;
  double2* trow;
  stage_layout<EPI>(ring, bar0, trow);
  // the previous stage's grid has completed; its writes are visible
  if (!stage_body<SCH, MODE, EPI>(a, ring, bar0, trow, [] { pdl_wait(); }, blockIdx.x))
    return;  // frozen
  // let the next stage's grid launch once this warp's rows are done (measured:
  // triggering at kernel start lets the next grid's waiting blocks take SM
  // slots early and costs 12 % at C5; triggering here gains 3-5 % on the
  // launch-bound small grids and is neutral at C5)
  pdl_trigger();
  if (a.tick != nullptr)
    launch_ticket(a.tick, a.flag, (a.px.on_lo | a.px.on_hi) ? a.px.epoch : nullptr,
                  (unsigned long long)gridDim.x * (blockDim.x >> 5));
}

// false: the state is frozen (an earlier step blew up) and nothing was done.
// ring / bar0 / trow: this warp's shared memory; wait_in(): returns once the
// stage's inputs written by other warps or grids are visible; bid: this
// block's index in the stage's launch (blockIdx.x, or the block's index
// within its slab in the peer emulation kernel, hwg_peer_emu.cu).
template <int SCH, int MODE, int EPI, class WaitIn>
__device__ __forceinline__ bool stage_body(const StageArgs& a, unsigned char* ring, uint32_t bar0,
                                           double2* trow, WaitIn&& wait_in, int bid) {
  using Wn = Win<SCH>;
  using SlotT = Slot<EPI>;
  constexpr int SL = Wn::SL, PL = Wn::PL, R = Wn::R, SW = Wn::SW, PW = Wn::PW;
  constexpr int IL = Wn::IL, IW = Wn::IW, S = SlotT::S, SB = SlotT::BYTES;
  constexpr bool CHECK = EPI == EPI_RK3C || EPI == EPI_RK104_10;
  extern __shared__ __align__(128) unsigned char smem[];
  const int lane = threadIdx.x & 31;
  const int wib = threadIdx.x >> 5;
  const int wpb = blockDim.x >> 5;                     // warps per block (1, 2 or 4)
  const int gw = bid * wpb + wib;
  const int chunk = gw % a.nchunks;
  const int range = gw / a.nchunks;
  const bool live = range < a.nranges;  // else the whole warp only takes its ticket
  const int span = a.row_hi - a.row_lo;
  const int jb = a.row_lo + (int)((long long)range * span / a.nranges);
  const int je = a.row_lo + (int)((long long)(range + 1) * span / a.nranges);
  const int k0 = chunk << 5;
  const int k = k0 + lane;
  const int nt = a.nt, n = a.n;
  const bool active = k < nt;
  const ptrdiff_t rs = (ptrdiff_t)a.rs;    // state row pitch (double2)
  const ptrdiff_t crs = (ptrdiff_t)a.crs;  // coefficient row pitch
  // theta halo: lanes 0,1 hold columns k0-2, k0-1; lanes 30,31 hold k0+32, k0+33
  const bool has_h = lane < 2 || lane >= 30;
  bool hflip;
  const int hoff = psi_off(reflect_col(lane < 2 ? k0 - 2 + lane : k0 + 2 + lane, nt, hflip,
                                       a.negpar));
  // idle lanes past the south pole publish the parity image of lane wsrc
  const bool pole_chunk = k0 + 32 > nt;
  bool wflip;
  const int wsrc = reflect_col(k, nt, wflip, a.negpar) - k0;

  const double2* xblk = a.x + chunk * kStateBlk;         // this chunk's block at row 0
  const double2* cblk = a.coef + chunk * kCoefBlk;

  // lane 0: the copies of iteration j into slot s.  The coefficient block
  // does not depend on the previous stage; the state blocks do.
  auto issue_coef = [&](int s, int j) {  // before pdl_wait: bytes expected, no arrival
    HWG_CHK(j >= 0 && j < n && chunk < a.nchunks);
    const uint32_t bar = bar0 + s * 8;
    mbar_expect_tx_only(bar, kCoefBlk * 16);
    bulk_g2s(smem_u32(ring + (size_t)s * SB) + SlotT::COEF, cblk + j * crs, kCoefBlk * 16, bar);
  };
  auto issue_state = [&](int s, int j, bool with_coef) {
    const uint32_t bar = bar0 + s * 8;
    const uint32_t dst = smem_u32(ring + (size_t)s * SB);
    const int rn = j + 1 + R;
    const bool st = (j + 1 < je) && !(rn >= n && a.phys_hi);
    const uint32_t bytes =
        SlotT::BYTES - (st ? 0 : kStateBlk * 16) - (with_coef ? 0 : kCoefBlk * 16);
    mbar_expect_tx(bar, bytes);  // + the arrival that completes the phase
    HWG_CHK(j >= 0 && j < n);
    HWG_CHK(!st || in_reg(xblk + rn * rs, a.x, rs, n, kStateBlk));
    HWG_CHK(!SlotT::HAS_A || in_reg(a.ua + j * rs + chunk * kStateBlk, a.ua, rs, n, kStateBlk));
    HWG_CHK(!SlotT::HAS_BG || (in_reg(a.ub + j * rs + chunk * kStateBlk, a.ub, rs, n, kStateBlk) &&
                               in_reg(a.ug + j * rs + chunk * kStateBlk, a.ug, rs, n, kStateBlk)));
    if (with_coef) bulk_g2s(dst + SlotT::COEF, cblk + j * crs, kCoefBlk * 16, bar);
    if (st) bulk_g2s(dst + SlotT::XN, xblk + rn * rs, kStateBlk * 16, bar);
    const ptrdiff_t o = j * rs + chunk * kStateBlk;
    if (SlotT::HAS_A) bulk_g2s(dst + SlotT::A, a.ua + o, kStateBlk * 16, bar);
    if (SlotT::HAS_BG) {
      bulk_g2s(dst + SlotT::B, a.ub + o, kStateBlk * 16, bar);
      bulk_g2s(dst + SlotT::G, a.ug + o, kStateBlk * 16, bar);
    }
  };
  // the row loop's refill of row jr: the same copies with running pointers
  // (advanced by one row each iteration) instead of per-row 64-bit products
  // (+1-2 % at C2, +1.5 % sustained, neutral at C5 burst;
  // profiles/r02_runptr_ab.txt)
  auto issue_row = [&](int s, int jr, const double2* csrc, const double2* xsrc, ptrdiff_t o) {
    const uint32_t bar = bar0 + s * 8;
    const uint32_t dst = smem_u32(ring + (size_t)s * SB);
    const int rn = jr + 1 + R;
    const bool st = (jr + 1 < je) && !(rn >= n && a.phys_hi);
    mbar_expect_tx(bar, SlotT::BYTES - (st ? 0 : kStateBlk * 16));
    HWG_CHK(jr >= 0 && jr < n && csrc == cblk + jr * crs && xsrc == xblk + rn * rs);
    HWG_CHK(!st || in_reg(xsrc, a.x, rs, n, kStateBlk));
    bulk_g2s(dst + SlotT::COEF, csrc, kCoefBlk * 16, bar);
    if (st) bulk_g2s(dst + SlotT::XN, xsrc, kStateBlk * 16, bar);
    if (SlotT::HAS_A) bulk_g2s(dst + SlotT::A, a.ua + o, kStateBlk * 16, bar);
    if (SlotT::HAS_BG) {
      bulk_g2s(dst + SlotT::B, a.ub + o, kStateBlk * 16, bar);
      bulk_g2s(dst + SlotT::G, a.ug + o, kStateBlk * 16, bar);
    }
  };
  const int nq = live ? (je - jb < S ? je - jb : S) : 0;  // slots primed
  // ---- prologue, overlapping the previous stage's tail (programmatic launch)
  if (lane == 0 && live) {
    for (int s = 0; s < S; ++s) mbar_init(bar0 + s * 8, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    // the ring may have been read by an earlier stage of the same launch
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    for (int q = 0; q < nq; ++q) issue_coef(q, jb + q);
  }
  wait_in();
  if (a.flag != nullptr && *(volatile unsigned long long*)a.flag != 0ull) {  // frozen
    if (lane == 0)
      for (int q = 0; q < nq; ++q) {  // drain the coefficient copies before exiting
        mbar_arrive(bar0 + q * 8);
        mbar_wait(bar0 + q * 8, 0);
      }
    // a frozen slab still releases its neighbours for this stage (no data)
    if (bid == 0 && threadIdx.x == 0 && (a.px.on_lo | a.px.on_hi)) {
      if (a.px.on_lo) peer_signal(a.px.sig_lo, (unsigned long long)a.nchunks);
      if (a.px.on_hi) peer_signal(a.px.sig_hi, (unsigned long long)a.nchunks);
      *a.px.epoch += 1ull;
    }
    return false;
  }
  if (a.bump && bid == 0 && threadIdx.x == 0) a.flag[2] += 1ull;  // step counter
  if (!live) return true;
  // boundary ranges: wait for the neighbours' halo rows of this stage
  if ((a.px.on_lo && range == 0) | (a.px.on_hi && range == a.nranges - 1))
    peer_wait_halos(a.px.wait, a.px.epoch, a.flag, a.nchunks, a.px.timeout_ns,
                    range == 0 && a.px.on_lo, range == a.nranges - 1 && a.px.on_hi);
  if (lane == 0)
    for (int q = 0; q < nq; ++q) issue_state(q, jb + q, false);
  __syncwarp();

  const double2* xps = xblk + lane;        // this lane's Psi at row 0
  const double2* xpi = xblk + 32 + lane;   // this lane's pi at row 0

  // ---- initial rows jb - IL .. jb + R (ghosts synthesised at the excision end)
  double2 ips[Wn::IA], ipi[Wn::IA];
  // rows -IL .. 3 of the excision end when this range starts within IL rows
  // of it: gs[IL + r] = row r, ghosts by the reference's recurrence
  // (t = 1, 2, ... from rows 0..3)
  const bool lo_ghosts = a.phys_lo && jb < IL;
  double2 gs[IL + 4], gp[IL + 4];
  if (lo_ghosts) {
#pragma unroll
    for (int m = 0; m < 4; ++m) {
      HWG_CHK(in_reg(xps + m * rs, a.x, rs, n, 1) && in_reg(xpi + m * rs, a.x, rs, n, 1));
      gs[IL + m] = __ldcg(xps + m * rs);
      gp[IL + m] = __ldcg(xpi + m * rs);
    }
#pragma unroll
    for (int t = 1; t <= IL; ++t) {
      gs[IL - t] = cubic(gs[IL - t + 1], gs[IL - t + 2], gs[IL - t + 3], gs[IL - t + 4]);
      gp[IL - t] = cubic(gp[IL - t + 1], gp[IL - t + 2], gp[IL - t + 3], gp[IL - t + 4]);
    }
  }
#pragma unroll
  for (int m = 0; m < IW; ++m) {
    const int r = jb - IL + m;
    if (lo_ghosts && r < 4) {
      ips[m] = gs[IL + r];
      ipi[m] = gp[IL + r];
    } else if (m >= 4 && r >= n && a.phys_hi) {  // scri continuation (r >= n implies m >= 4)
      ips[m] = cubic(ips[m - 1], ips[m - 2], ips[m - 3], ips[m - 4]);
      ipi[m] = cubic(ipi[m - 1], ipi[m - 2], ipi[m - 3], ipi[m - 4]);
    } else {
      HWG_CHK(in_reg(xps + r * rs, a.x, rs, n, 1) && in_reg(xpi + r * rs, a.x, rs, n, 1));
      ips[m] = __ldcg(xps + r * rs);
      ipi[m] = __ldcg(xpi + r * rs);
    }
  }
  double2 wps[SW], wpi[PW];
#pragma unroll
  for (int m = 0; m < SW; ++m) wps[m] = ips[IL - SL + m];
#pragma unroll
  for (int m = 0; m < PW; ++m) wpi[m] = ipi[IL - PL + m];

  const double cot = __ldg(a.cot + k);
  // carried interface values F(j - 1/2)
  double2 fps = make_double2(0.0, 0.0), fpi = fps;
  bool opi = __ldg(&cblk[jb * crs + lane].y) < 0.0;  // orientation of fpi (true = minus)
  if (SCH != FD6KO) {
    fps = iface2_at<SCH, MODE, IL>(ips, true, -1, a);
    fpi = iface2_at<SCH, MODE, IL>(ipi, opi, -1, a);
  }

  bool bad = false;
  // theta halo, software-pipelined one row ahead (4 lanes)
  const double2* hrow = a.x + hoff + (ptrdiff_t)jb * rs;
  HWG_CHK(!has_h || in_reg(hrow, a.x, rs, n, 1));
  const double hsgn = hflip ? -1.0 : 1.0;  // the parity image's sign (exact: -x == x * -1)
  double2 hn = has_h ? ld2(hrow) : make_double2(0.0, 0.0);
  int slot = 0;
  uint32_t parity = 0;
  // rows per unrolled iteration: 2 lets the register windows rotate with half
  // the moves (measured +1.5-4 % at 168 registers; 3 and 4 are slower)
#ifdef HWG_UNROLL
  constexpr int kUnroll = HWG_UNROLL;
#else
  constexpr int kUnroll = SCH == WENO5 ? 2 : 1;
#endif
  // running sources of the refill S rows ahead (issue_row)
  const double2* iss_c = cblk + (ptrdiff_t)(jb + S) * crs;
  const double2* iss_x = xblk + (ptrdiff_t)(jb + S + 1 + R) * rs;
  ptrdiff_t iss_o = (ptrdiff_t)(jb + S) * rs + chunk * kStateBlk;
#pragma unroll kUnroll
  for (int j = jb; j < je; ++j) {
    const unsigned char* sl = ring + (size_t)slot * SB;
    const double2* sd = reinterpret_cast<const double2*>(sl) + lane;
    // software-pipelined one row ahead; the row after the range's last is a
    // valid (halo or interior) row of the register, so no range test — a
    // predicated load, and the parity sign applied at the store (-1.4 % warp
    // instructions, +1-2.5 % at C5 and C2, +1.3 % under the power cap)
    const double2 h = hn;
    hrow += rs;
    HWG_CHK(!has_h || in_reg(hrow, a.x, rs, n, 1));
    if (has_h) hn = ld2(hrow);
    mbar_wait(bar0 + slot * 8, parity);
    const double2 bl = sd[0];

    // ---- phase 1: radial derivatives
    double2 dps, dpi;
    if (SCH != FD6KO) {
      // Psi rows: right-biased everywhere (b <= 0; evolve.cpp:103-104)
      const double2 cs = iface2_at<SCH, MODE, SL>(wps, true, 0, a);
      // unscaled differences: 1/(6 drho) lives in the planes b, lam, w
      dps = make_double2(cs.x - fps.x, cs.y - fps.y);
      fps = cs;
      // pi rows: minus where lam < 0 (split_k rule, evolve.cpp:19-30, 105-110)
      const bool o = bl.y < 0.0;
      if (o != opi) {
        // start of a sub-row: fresh F(j - 1/2) in the new orientation
        if (!o && SCH == WENO5) {
          // plus at j - 1/2 needs row j - 3, outside the window
          double2 xx[PW + 1];
          HWG_CHK(j - 3 >= -kHalo);
          xx[0] = row_or_ghost(xpi, j - 3, rs, a.phys_lo);
#pragma unroll
          for (int m = 0; m < PW; ++m) xx[m + 1] = wpi[m];
          fpi = iface2_at<SCH, MODE, PL + 1>(xx, false, -1, a);
        } else {
          fpi = iface2_at<SCH, MODE, PL>(wpi, o, -1, a);
        }
        opi = o;
      }
      double2 pp;
      if (__all_sync(kFull, !o)) pp = iface2_at<SCH, MODE, PL>(wpi, false, 0, a);
      else pp = iface2_at<SCH, MODE, PL>(wpi, o, 0, a);
      dpi = make_double2(pp.x - fpi.x, pp.y - fpi.y);
      fpi = pp;
    } else {
      // FD6 (spatial.hpp:178-182): centred, no upwinding, all four rows
      auto fd6 = [&](double m3, double m2, double m1, double p1, double p2, double p3) {
        return fma(45.0, p1 - m1, fma(-9.0, p2 - m2, p3 - m3));  // 1/(60 drho) in the planes
      };
      constexpr int C = SL;
      dps = make_double2(
          fd6(wps[C - 3].x, wps[C - 2].x, wps[C - 1].x, wps[C + 1].x, wps[C + 2].x, wps[C + 3].x),
          fd6(wps[C - 3].y, wps[C - 2].y, wps[C - 1].y, wps[C + 1].y, wps[C + 2].y, wps[C + 3].y));
      dpi = make_double2(
          fd6(wpi[C - 3].x, wpi[C - 2].x, wpi[C - 1].x, wpi[C + 1].x, wpi[C + 2].x, wpi[C + 3].x),
          fd6(wpi[C - 3].y, wpi[C - 2].y, wpi[C - 1].y, wpi[C + 1].y, wpi[C + 2].y, wpi[C + 3].y));
    }

    // ---- phase 2: (d_thth + cot d_th) Psi (spatial.hpp:208-222)
    const double2 ps = wps[SL];
    double2 wv = ps;   // value this lane publishes to its theta neighbours
    if (pole_chunk) {  // warp-uniform
      double2 img = make_double2(__shfl_sync(kFull, ps.x, wsrc & 31),
                                 __shfl_sync(kFull, ps.y, wsrc & 31));
      // image column in the previous chunk (last chunk with one column)
      if (!active && (wsrc < 0 || wsrc > 31)) {
        HWG_CHK(in_reg(a.x + (ptrdiff_t)j * rs + psi_off(k0 + wsrc), a.x, rs, n, 1));
        img = ld2(a.x + (ptrdiff_t)j * rs + psi_off(k0 + wsrc));
      }
      if (!active) wv = wflip ? neg2(img) : img;
    }
    // the chunk's extended row E[i] = Psi(k0 - 2 + i), i < 36, in shared memory
    // (one store + four loads instead of 12 double shuffles and selects)
    trow[lane + 2] = wv;
    if (has_h) trow[lane < 2 ? lane : lane + 4] = make_double2(h.x * hsgn, h.y * hsgn);
    __syncwarp();
    const double2 m2 = trow[lane], m1 = trow[lane + 1], p1 = trow[lane + 3], p2 = trow[lane + 4];
    // 12 dth^2 (d_thth + cot d_th): the factor 1/(12 dth^2) is folded into
    // ath and cot carries dth (coefficient upload, hwg_solver.cu)
    const double d1R = fma(8.0, p1.x - m1.x, m2.x - p2.x);
    const double d1I = fma(8.0, p1.y - m1.y, m2.y - p2.y);
    const double d2R = fma(-30.0, ps.x, fma(16.0, m1.x + p1.x, -(m2.x + p2.x)));
    const double d2I = fma(-30.0, ps.y, fma(16.0, m1.y + p1.y, -(m2.y + p2.y)));
    const double angR = fma(cot, d1R, d2R);
    const double angI = fma(cot, d1I, d2I);

    // ---- phase 3: pointwise assembly (evolve.cpp:149-167)
    const double2 cw = sd[32], cbt = sd[64], ccf = sd[96];
    const double ath = reinterpret_cast<const double*>(sl + kCoefAth * 16)[lane];
    const double2 pv = wpi[PL];
    const double b = bl.x, lam = bl.y;
    double f0 = fma(-b, dps.x, pv.x);
    double f1 = fma(-b, dps.y, pv.y);
    double f2v = fma(ath, angR, fma(-ccf.y, ps.y, fma(ccf.x, ps.x, fma(-cbt.y, pv.y,
                 fma(cbt.x, pv.x, fma(-cw.y, dps.y, fma(cw.x, dps.x, -lam * dpi.x)))))));
    double f3 = fma(ath, angI, fma(ccf.y, ps.x, fma(ccf.x, ps.y, fma(cbt.y, pv.x,
                fma(cbt.x, pv.y, fma(cw.y, dps.x, fma(cw.x, dps.y, -lam * dpi.y)))))));
    if (SCH == FD6KO) {
      // KO8 (spatial.hpp:184-191), subtracted from all four rows (evolve.cpp:169-176)
      auto ko8 = [&](double u4m, double u3m, double u2m, double u1m, double u0, double u1p,
                     double u2p, double u3p, double u4p) {
        double d8 = fma(70.0, u0, fma(-56.0, u1m + u1p, fma(28.0, u2m + u2p,
                        fma(-8.0, u3m + u3p, u4m + u4p))));
        return d8 * a.ko;
      };
      f0 -= ko8(wps[0].x, wps[1].x, wps[2].x, wps[3].x, wps[4].x, wps[5].x, wps[6].x, wps[7].x, wps[8].x);
      f1 -= ko8(wps[0].y, wps[1].y, wps[2].y, wps[3].y, wps[4].y, wps[5].y, wps[6].y, wps[7].y, wps[8].y);
      f2v -= ko8(wpi[0].x, wpi[1].x, wpi[2].x, wpi[3].x, wpi[4].x, wpi[5].x, wpi[6].x, wpi[7].x, wpi[8].x);
      f3 -= ko8(wpi[0].y, wpi[1].y, wpi[2].y, wpi[3].y, wpi[4].y, wpi[5].y, wpi[6].y, wpi[7].y, wpi[8].y);
    }

    // ---- RK epilogue (timestep.hpp:61-70, 84-108): the reference's
    // combinations, with its multiply-adds fused
    double2 ops, opv;
    if (EPI == EPI_RHS) {
      ops = make_double2(f0, f1); opv = make_double2(f2v, f3);
    } else if (EPI == EPI_AXPY) {
      ops = make_double2(fma(a.cg, f0, ps.x), fma(a.cg, f1, ps.y));
      opv = make_double2(fma(a.cg, f2v, pv.x), fma(a.cg, f3, pv.y));
    } else {
      const double2* sa = reinterpret_cast<const double2*>(sl + SlotT::A) + lane;
      const double2 aps = sa[0], api = sa[32];
      if (EPI == EPI_RK3 || EPI == EPI_RK3C) {
        ops = make_double2(fma(a.ca, aps.x, a.cb * fma(a.cg, f0, ps.x)),
                           fma(a.ca, aps.y, a.cb * fma(a.cg, f1, ps.y)));
        opv = make_double2(fma(a.ca, api.x, a.cb * fma(a.cg, f2v, pv.x)),
                           fma(a.ca, api.y, a.cb * fma(a.cg, f3, pv.y)));
      } else if (EPI == EPI_RK104_5) {
        ops = make_double2(fma(a.cg, f0, fma(a.cb, ps.x, a.ca * aps.x)),
                           fma(a.cg, f1, fma(a.cb, ps.y, a.ca * aps.y)));
        opv = make_double2(fma(a.cg, f2v, fma(a.cb, pv.x, a.ca * api.x)),
                           fma(a.cg, f3, fma(a.cb, pv.y, a.ca * api.y)));
      } else {
        const double2* sb = reinterpret_cast<const double2*>(sl + SlotT::B) + lane;
        const double2* sg = reinterpret_cast<const double2*>(sl + SlotT::G) + lane;
        const double2 bps = sb[0], bpi = sb[32], gps = sg[0], gpi = sg[32];
        auto c10 = [&](double A, double B, double x, double G, double f) {
          return fma(a.cg, fma(a.cd, G, a.ce * f), fma(a.cc, x, fma(a.cb, B, a.ca * A)));
        };
        ops = make_double2(c10(aps.x, bps.x, ps.x, gps.x, f0), c10(aps.y, bps.y, ps.y, gps.y, f1));
        opv = make_double2(c10(api.x, bpi.x, pv.x, gpi.x, f2v), c10(api.y, bpi.y, pv.y, gpi.y, f3));
      }
    }
    if (active) {
      double2* ob = a.o + j * rs + chunk * kStateBlk + lane;
      HWG_CHK(j >= 0 && j < n && in_reg(ob, a.o, rs, n, 33));
      ob[0] = ops;
      ob[32] = opv;
      if (EPI == EPI_RK104_5) {
        double2* fb = a.f + j * rs + chunk * kStateBlk + lane;
        HWG_CHK(in_reg(fb, a.f, rs, n, 33));
        fb[0] = make_double2(f0, f1);
        fb[32] = make_double2(f2v, f3);
      }
      if (CHECK) {
        // state_admissible (evolve.cpp:217-235): NaN or |u| > 1e30
        bad |= !(fabs(ops.x) <= 1e30) || !(fabs(ops.y) <= 1e30) || !(fabs(opv.x) <= 1e30) ||
               !(fabs(opv.y) <= 1e30);
      }
    }

    // ---- slide the windows
    const int rn = j + 1 + R;
#pragma unroll
    for (int m = 0; m < SW - 1; ++m) wps[m] = wps[m + 1];
#pragma unroll
    for (int m = 0; m < PW - 1; ++m) wpi[m] = wpi[m + 1];
    if (rn >= n && a.phys_hi) {
      wps[SW - 1] = cubic(wps[SW - 2], wps[SW - 3], wps[SW - 4], wps[SW - 5]);
      wpi[PW - 1] = cubic(wpi[PW - 2], wpi[PW - 3], wpi[PW - 4], wpi[PW - 5]);
    } else {
      const double2* sx = reinterpret_cast<const double2*>(sl + SlotT::XN) + lane;
      wps[SW - 1] = sx[0];
      wpi[PW - 1] = sx[32];
    }
    // ---- release the slot and refill it S rows ahead
    __syncwarp();
    // one elected lane issues the next row's copies: with elect.sync the
    // compiler knows a single lane runs the block (−2 % at C2, +1–1.5 % at C5
    // and sustained against `lane == 0`, profiles/r02_elect_ab.txt)
    if (j + S < je && elect_one()) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      issue_row(slot, j + S, iss_c, iss_x, iss_o);
    }
    iss_c += crs;
    iss_x += rs;
    iss_o += rs;
    if (++slot == S) { slot = 0; parity ^= 1u; }
  }
  if ((a.px.on_lo && jb == 0) | (a.px.on_hi && je == n))
    peer_push_halos(a.o, a.px.o_lo, a.px.o_hi, a.px.sig_lo, a.px.sig_hi, rs, n, nt,
                    a.px.h, chunk, a.px.on_lo && jb == 0, a.px.on_hi && je == n);
  if (CHECK && __any_sync(kFull, bad) && lane == 0) {
    atomicExch(a.flag + 1, a.step >= 0 ? (unsigned long long)a.step : a.flag[2]);
    // published by the launch's last warp (tick) so no block of this launch
    // sees a half-frozen state
    atomicOr(a.flag + (a.tick != nullptr || a.defer ? 3 : 0), 1ull);
  }
  return true;
}

}  // namespace hwg
