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
// Device layout: theta fastest.  A state register is two
// planes of double2 — Psi = (Psi_R, Psi_I) and pi = (pi_R, pi_I) — with rows
// j in [-kHalo, n + kHalo) and a row pitch ntp = ntheta rounded up to 32.
// Coefficients are double2 planes (b, lam), (w_re, w_im), (bt_re, bt_im),
// (c_re, c_im) plus a double plane ath, rows [0, n).
//
// Work decomposition: a warp owns a 32-column theta chunk and a contiguous
// range of rows; each lane owns one theta column and marches along rho with a
// register window of the stencil rows, so every state value is loaded from
// HBM once (plus 2 x halo rows per range).  Theta neighbours come from warp
// shuffles (parity-reflected at the poles, evolve.cpp:59-70); only the two
// lanes at each warp edge load a neighbour column.  Radial ghosts at the
// physical ends are synthesised in registers with the reference's cubic
// recurrence (evolve.cpp:45-57); slab ends read halo rows.
//
// Arithmetic: compiled with -fmad=false; every fused multiply-add below is an
// explicit fma(), so the result of an interface does not depend on where it
// is computed (slab boundaries reproduce the single-GPU result bitwise).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace hwg {

#ifndef HWG_MINB
#define HWG_MINB 4  // resident blocks per SM (16 warps): caps registers at 128
#endif
#ifndef HWG_RING
#define HWG_RING 3  // bulk-copy ring depth (rows in flight + 1) per warp
#endif

constexpr int kHalo = 4;          // halo rows per side (KO8 needs 4)
constexpr int kWarpsPerBlock = 4;
constexpr unsigned kFull = 0xffffffffu;

enum SchemeId { WENO5 = 0, WENO3 = 1, FD6KO = 2 };
enum ModeId { F64 = 0, MIXED = 1 };
enum EpiId {
  EPI_RHS = 0,       // o = f                                       (EvolutionRhs)
  EPI_AXPY = 1,      // o = x + g f                                 (rk33 stage 1, rk104 i)
  EPI_RK3 = 2,       // o = a A + b (x + g f)                       (rk33 stages 2, 3)
  EPI_RK104_5 = 3,   // o = a A + b x + g f ; F4 = f                (rk104 stage 5)
  EPI_RK104_10 = 4   // o = a A + b B + c x + g (d G + e f)         (rk104 stage 10)
};

struct StageArgs {
  int n, nt, ntp;
  int phys_lo, phys_hi;            // slab holds the excision / scri end
  int nchunks, nranges;
  int linear;                      // eps = inf: frozen linear weights
  int negpar;                      // theta parity (-1)^(m+s) == -1
  int check;                       // admissibility scan in this stage
  long long step;                  // blowup_step recorded if the scan fails
  double eps4;                     // fp64 weights: 4 eps (scaled indicators)
  double eps;                      // fp64 weno3
  float epsf;                      // fp32 weights: eps demoted
  double iscale;                   // radial derivative scale
  double inv1, inv2;               // theta: 1/(12 dth), 1/(12 dth^2)
  double ko;                       // KO8: sigma / (256 drho)
  double ca, cb, cc, cg, cd, ce;   // epilogue coefficients
  // state planes, pointers at row 0 (halo rows at negative offsets)
  const double2* xpsi; const double2* xpi;   // stencil input u_k
  const double2* apsi; const double2* api;   // u_n
  const double2* bpsi; const double2* bpi;   // u^(4)
  const double2* gpsi; const double2* gpi;   // F(u^(4))
  double2* opsi; double2* opi;               // output
  double2* fpsi; double2* fpi;               // F store (rk104 stage 5)
  // coefficient planes, rows [0, n)
  const double2* cbl; const double2* cw; const double2* cbt; const double2* ccf;
  const double* cath; const double* cot;
  unsigned long long* flag;                  // [0] blown, [1] blowup step
};

__device__ __forceinline__ double2 ld2(const double2* p) { return __ldg(p); }

__device__ __forceinline__ double2 neg2(double2 v) { return make_double2(-v.x, -v.y); }

// reference cubic continuation (defined below), used by row_or_ghost
__device__ __forceinline__ double2 cubic(double2 a, double2 b, double2 c, double2 d);

// state row r of one plane column; rows < 0 of the slab holding the
// excision end are the reference's cubic ghosts (rare path: orientation switch)
__device__ __noinline__ double2 row_or_ghost(const double2* col, int r, ptrdiff_t ntp, int phys_lo) {
  if (r >= 0 || !phys_lo) return __ldg(col + r * ntp);
  double2 g[8];
  for (int m = 0; m < 4; ++m) g[4 + m] = __ldg(col + m * ntp);
  for (int t = 1; t <= -r; ++t) g[4 - t] = cubic(g[4 - t + 1], g[4 - t + 2], g[4 - t + 3], g[4 - t + 4]);
  return g[4 + r];
}

// reference cubic continuation p[-t] = 4p[-t+1] - 6p[-t+2] + 4p[-t+3] - p[-t+4]
// (evolve.cpp:48-50), same evaluation order
__device__ __forceinline__ double cubic1(double a, double b, double c, double d) {
  return 4.0 * a - 6.0 * b + 4.0 * c - d;
}
__device__ __forceinline__ double2 cubic(double2 a, double2 b, double2 c, double2 d) {
  return make_double2(cubic1(a.x, b.x, c.x, d.x), cubic1(a.y, b.y, c.y, d.y));
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
// WENO5-JS interface value (spatial.hpp:29-92) on the oriented window
// f0..f4, returned WITHOUT the 1/6 factor (folded into iscale).
//
// fp64 weights: alpha_k = d_k/(eps + IS_k)^2 normalised; with the indicators
// scaled by 4 (IS' = 13/3 t^2 + s^2, eps' = 4 eps) the weights are
// w_k = d_k prod_{i!=k} e_i^2 / sum(...), so one reciprocal replaces the
// reference's five divisions (weights and renormalisation, spatial.hpp:58-90).
__device__ __forceinline__ double weno5_f64(double f0, double f1, double f2, double f3,
                                            double f4, double eps4, int linear) {
  double n0, n1, n2;
  if (linear) {
    n0 = 1.0; n1 = 6.0; n2 = 3.0;
  } else {
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
    n0 = q1 * q2;
    n1 = 6.0 * (q0 * q2);
    n2 = 3.0 * (q0 * q1);
  }
  double c0 = fma(11.0, f2, fma(-7.0, f1, 2.0 * f0));
  double c1 = fma(2.0, f3, fma(5.0, f2, -f1));
  double c2 = fma(5.0, f3, fma(2.0, f2, -f4));
  double num = fma(n2, c2, fma(n1, c1, n0 * c0));
  return num * drcp((n0 + n1) + n2);
}

// Mixed mode (the paper's): window demoted to fp32, smoothness indicators and
// nonlinear weights in fp32 (spatial.hpp:29-65 with TW = float), promoted and
// renormalised in fp64 work precision (:84-90), fp64 candidate stencils.
__device__ __forceinline__ double weno5_mixed(double f0, double f1, double f2, double f3,
                                              double f4, float eps, int linear) {
  float w0, w1, w2;
  if (linear) {
    w0 = 0.1f; w1 = 0.6f; w2 = 0.3f;
  } else {
    const float g0 = (float)f0, g1 = (float)f1, g2 = (float)f2, g3 = (float)f3,
                g4 = (float)f4;
    const float c1312 = 13.0f / 12.0f, qt = 0.25f;
    float t = fmaf(-2.0f, g1, g0) + g2;
    float s = fmaf(3.0f, g2, fmaf(-4.0f, g1, g0));
    float e0 = eps + fmaf(c1312 * t, t, qt * s * s);
    t = fmaf(-2.0f, g2, g1) + g3;
    s = g1 - g3;
    float e1 = eps + fmaf(c1312 * t, t, qt * s * s);
    t = fmaf(-2.0f, g3, g2) + g4;
    s = fmaf(3.0f, g2, fmaf(-4.0f, g3, g4));
    float e2 = eps + fmaf(c1312 * t, t, qt * s * s);
    float a0 = 0.1f * frcp(e0 * e0);
    float a1 = 0.6f * frcp(e1 * e1);
    float a2 = 0.3f * frcp(e2 * e2);
    float inv = frcp((a0 + a1) + a2);
    w0 = a0 * inv; w1 = a1 * inv; w2 = a2 * inv;
  }
  const double W0 = (double)w0, W1 = (double)w1, W2 = (double)w2;
  double c0 = fma(11.0, f2, fma(-7.0, f1, 2.0 * f0));
  double c1 = fma(2.0, f3, fma(5.0, f2, -f1));
  double c2 = fma(5.0, f3, fma(2.0, f2, -f4));
  double num = fma(W2, c2, fma(W1, c1, W0 * c0));
  return num * drcp((W0 + W1) + W2);
}

template <int MODE>
__device__ __forceinline__ double weno5(double f0, double f1, double f2, double f3, double f4,
                                        const StageArgs& a) {
  if (MODE == F64) return weno5_f64(f0, f1, f2, f3, f4, a.eps4, a.linear);
  return weno5_mixed(f0, f1, f2, f3, f4, a.epsf, a.linear);
}

// WENO3 interface (spatial.hpp:94-130), without the 1/2 (folded into iscale)
template <int MODE>
__device__ __forceinline__ double weno3(double f0, double f1, double f2, const StageArgs& a) {
  double n0, n1;
  if (a.linear) {
    n0 = 1.0; n1 = 2.0;
  } else if (MODE == F64) {
    double d0 = f1 - f0, d1 = f2 - f1;
    double e0 = fma(d0, d0, a.eps), e1 = fma(d1, d1, a.eps);
    n0 = e1 * e1;
    n1 = 2.0 * (e0 * e0);
  } else {
    float g0 = (float)f0, g1 = (float)f1, g2 = (float)f2;
    float d0 = g1 - g0, d1 = g2 - g1;
    float e0 = fmaf(d0, d0, a.epsf), e1 = fmaf(d1, d1, a.epsf);
    float x0 = (1.0f / 3.0f) * frcp(e0 * e0);
    float x1 = (2.0f / 3.0f) * frcp(e1 * e1);
    float inv = frcp(x0 + x1);
    n0 = (double)(x0 * inv);
    n1 = (double)(x1 * inv);
  }
  double q0 = fma(3.0, f1, -f0);
  double q1 = f1 + f2;
  return fma(n1, q1, n0 * q0) * drcp(n0 + n1);
}

// interface value of one oriented window for either scheme (w[] = window
// rows j - L .. j + R, C = index of row j); minus = right-biased mirror.
template <int SCH, int MODE, int C>
__device__ __forceinline__ double iface_at(const double* w, bool minus, int shift,
                                           const StageArgs& a) {
  // interface j + 1/2 + shift
  const int c = C + shift;
  if (SCH == WENO5) {
    return minus ? weno5<MODE>(w[c + 3], w[c + 2], w[c + 1], w[c], w[c - 1], a)
                 : weno5<MODE>(w[c - 2], w[c - 1], w[c], w[c + 1], w[c + 2], a);
  }
  return minus ? weno3<MODE>(w[c + 2], w[c + 1], w[c], a)
               : weno3<MODE>(w[c - 1], w[c], w[c + 1], a);
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
  static constexpr int IA = (IL + 4 > IW) ? IL + 4 : IW;  // init array (4 rows for the cubic)
};

__device__ __forceinline__ double2 shfl_up2(double2 v, int d) {
  return make_double2(__shfl_up_sync(kFull, v.x, d), __shfl_up_sync(kFull, v.y, d));
}
__device__ __forceinline__ double2 shfl_dn2(double2 v, int d) {
  return make_double2(__shfl_down_sync(kFull, v.x, d), __shfl_down_sync(kFull, v.y, d));
}

// parity reflection of a theta column across the poles (evolve.cpp:59-70)
__device__ __forceinline__ int reflect_col(int c, int nt, bool& flip, int negpar) {
  flip = false;
  if (c < 0) { c = -1 - c; flip = negpar; }
  else if (c >= nt) { c = 2 * nt - 1 - c; flip = negpar; }
  if (c < 0 || c >= nt) { c = 0; flip = false; }  // only for lanes far outside tiny grids
  return c;
}

// ---------------------------------------------------------------------------
// Bulk-copy (TMA engine) row ring.  Each warp owns S slots of shared memory;
// slot s holds, for one iteration j: the pointwise data of row j (the 9
// coefficient values as 4 double2 planes + ath, u_n, u^(4), F(u^(4)) as the
// epilogue needs) and the stencil-input row j + 1 + R that enters the
// register window at the end of the iteration.  Lane 0 issues the row's
// cp.async.bulk copies S iterations ahead; an mbarrier per slot completes on
// the transferred byte count.  The warp's lanes then read their own column
// from shared memory, so the prefetch costs no registers.
template <int EPI>
struct Slot {
  static constexpr int ROWB = 32 * 16;                 // one double2 row chunk
  static constexpr int BL = 0, CW = ROWB, CBT = 2 * ROWB, CCF = 3 * ROWB;
  static constexpr int XPS = 4 * ROWB, XPI = 5 * ROWB;  // next stencil row
  static constexpr int ATH = 6 * ROWB;                  // 32 doubles
  static constexpr int BASE = ATH + 32 * 8;
  static constexpr bool HAS_A = EPI == EPI_RK3 || EPI == EPI_RK104_5 || EPI == EPI_RK104_10;
  static constexpr bool HAS_BG = EPI == EPI_RK104_10;
  static constexpr int APS = BASE, API = BASE + ROWB;
  static constexpr int BPS = BASE + 2 * ROWB, BPI = BASE + 3 * ROWB;
  static constexpr int GPS = BASE + 4 * ROWB, GPI = BASE + 5 * ROWB;
  static constexpr int BYTES = BASE + (HAS_A ? 2 * ROWB : 0) + (HAS_BG ? 4 * ROWB : 0);
  static constexpr int S = HAS_BG ? 2 : HWG_RING;       // ring depth
};

template <int EPI>
constexpr size_t stage_smem_bytes() {
  return (size_t)kWarpsPerBlock * Slot<EPI>::S * (Slot<EPI>::BYTES + 8);
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

template <int SCH, int MODE, int EPI>
__global__ void __launch_bounds__(kWarpsPerBlock * 32, HWG_MINB)
stage_kernel(const StageArgs a) {
  if (a.flag != nullptr && *(volatile unsigned long long*)a.flag != 0ull) return;  // frozen
  using Wn = Win<SCH>;
  using SlotT = Slot<EPI>;
  constexpr int SL = Wn::SL, PL = Wn::PL, R = Wn::R, SW = Wn::SW, PW = Wn::PW;
  constexpr int IL = Wn::IL, IW = Wn::IW, S = SlotT::S, SB = SlotT::BYTES;
  extern __shared__ __align__(128) unsigned char smem[];
  const int lane = threadIdx.x & 31;
  const int wib = threadIdx.x >> 5;
  const int gw = blockIdx.x * kWarpsPerBlock + wib;
  const int chunk = gw % a.nchunks;
  const int range = gw / a.nchunks;
  if (range >= a.nranges) return;                       // whole warp
  const int jb = (int)((long long)range * a.n / a.nranges);
  const int je = (int)((long long)(range + 1) * a.n / a.nranges);
  const int k0 = chunk << 5;
  const int k = k0 + lane;
  const int nt = a.nt, n = a.n;
  const bool active = k < nt;
  const ptrdiff_t ntp = a.ntp;
  const int kc = active ? k : nt - 1;
  // theta halo: lanes 0,1 hold columns k0-2, k0-1; lanes 30,31 hold k0+32, k0+33
  const bool has_h = lane < 2 || lane >= 30;
  bool hflip;
  const int hcol = reflect_col(lane < 2 ? k0 - 2 + lane : k0 + 2 + lane, nt, hflip, a.negpar);
  // idle lanes past the south pole publish the parity image of lane refl
  const bool pole_chunk = k0 + 32 > nt;
  bool wflip;
  const int wsrc = reflect_col(k, nt, wflip, a.negpar) - k0;

  unsigned char* ring = smem + (size_t)wib * S * SB;
  const uint32_t bar0 = smem_u32(smem + (size_t)kWarpsPerBlock * S * SB) + wib * S * 8;

  // lane 0: issue the copies of iteration j into slot s
  auto issue = [&](int s, int j) {
    const uint32_t bar = bar0 + s * 8;
    const uint32_t dst = smem_u32(ring + (size_t)s * SB);
    const int rn = j + 1 + R;
    const bool st = (j + 1 < je) && !(rn >= n && a.phys_hi);
    const uint32_t bytes = SlotT::BASE - (st ? 0 : 2 * SlotT::ROWB) +
                           (SlotT::HAS_A ? 2 * SlotT::ROWB : 0) +
                           (SlotT::HAS_BG ? 4 * SlotT::ROWB : 0);
    mbar_expect_tx(bar, bytes);
    const ptrdiff_t o = (ptrdiff_t)j * ntp + k0;
    bulk_g2s(dst + SlotT::BL, a.cbl + o, SlotT::ROWB, bar);
    bulk_g2s(dst + SlotT::CW, a.cw + o, SlotT::ROWB, bar);
    bulk_g2s(dst + SlotT::CBT, a.cbt + o, SlotT::ROWB, bar);
    bulk_g2s(dst + SlotT::CCF, a.ccf + o, SlotT::ROWB, bar);
    bulk_g2s(dst + SlotT::ATH, a.cath + o, 32 * 8, bar);
    if (st) {
      const ptrdiff_t os = (ptrdiff_t)rn * ntp + k0;
      bulk_g2s(dst + SlotT::XPS, a.xpsi + os, SlotT::ROWB, bar);
      bulk_g2s(dst + SlotT::XPI, a.xpi + os, SlotT::ROWB, bar);
    }
    if (SlotT::HAS_A) {
      bulk_g2s(dst + SlotT::APS, a.apsi + o, SlotT::ROWB, bar);
      bulk_g2s(dst + SlotT::API, a.api + o, SlotT::ROWB, bar);
    }
    if (SlotT::HAS_BG) {
      bulk_g2s(dst + SlotT::BPS, a.bpsi + o, SlotT::ROWB, bar);
      bulk_g2s(dst + SlotT::BPI, a.bpi + o, SlotT::ROWB, bar);
      bulk_g2s(dst + SlotT::GPS, a.gpsi + o, SlotT::ROWB, bar);
      bulk_g2s(dst + SlotT::GPI, a.gpi + o, SlotT::ROWB, bar);
    }
  };
  if (lane == 0) {
    for (int s = 0; s < S; ++s) mbar_init(bar0 + s * 8, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    for (int q = 0; q < S && jb + q < je; ++q) issue(q, jb + q);
  }
  __syncwarp();

  const double2* xps = a.xpsi + kc;
  const double2* xpi = a.xpi + kc;

  // ---- initial rows jb - IL .. jb + R (ghosts synthesised at the excision end)
  double2 ips[Wn::IA], ipi[Wn::IA];
  if (a.phys_lo && jb < IL) {
    // only jb == 0 happens (ranges are >= 8 rows)
#pragma unroll
    for (int m = 0; m < 4; ++m) {
      ips[IL + m] = ld2(xps + m * ntp);
      ipi[IL + m] = ld2(xpi + m * ntp);
    }
#pragma unroll
    for (int t = 1; t <= IL; ++t) {
      ips[IL - t] = cubic(ips[IL - t + 1], ips[IL - t + 2], ips[IL - t + 3], ips[IL - t + 4]);
      ipi[IL - t] = cubic(ipi[IL - t + 1], ipi[IL - t + 2], ipi[IL - t + 3], ipi[IL - t + 4]);
    }
#pragma unroll
    for (int m = IL + 4; m < IW; ++m) {
      ips[m] = ld2(xps + (m - IL) * ntp);
      ipi[m] = ld2(xpi + (m - IL) * ntp);
    }
  } else {
#pragma unroll
    for (int m = 0; m < IW; ++m) {
      const int r = jb - IL + m;
      if (r >= n && a.phys_hi) {
        ips[m] = cubic(ips[m - 1], ips[m - 2], ips[m - 3], ips[m - 4]);
        ipi[m] = cubic(ipi[m - 1], ipi[m - 2], ipi[m - 3], ipi[m - 4]);
      } else {
        ips[m] = ld2(xps + r * ntp);
        ipi[m] = ld2(xpi + r * ntp);
      }
    }
  }
  double2 wps[SW], wpi[PW];
#pragma unroll
  for (int m = 0; m < SW; ++m) wps[m] = ips[IL - SL + m];
#pragma unroll
  for (int m = 0; m < PW; ++m) wpi[m] = ipi[IL - PL + m];

  const double cot = __ldg(a.cot + kc);
  // carried interface values F(j - 1/2)
  double fpsR = 0.0, fpsI = 0.0, fpiR = 0.0, fpiI = 0.0;
  bool opi = __ldg(&a.cbl[(ptrdiff_t)jb * ntp + kc].y) < 0.0;  // true = minus
  if (SCH != FD6KO) {
    double r[IW], q[IW];
#pragma unroll
    for (int m = 0; m < IW; ++m) { r[m] = ips[m].x; q[m] = ips[m].y; }
    fpsR = iface_at<SCH, MODE, IL>(r, true, -1, a);
    fpsI = iface_at<SCH, MODE, IL>(q, true, -1, a);
#pragma unroll
    for (int m = 0; m < IW; ++m) { r[m] = ipi[m].x; q[m] = ipi[m].y; }
    fpiR = iface_at<SCH, MODE, IL>(r, opi, -1, a);
    fpiI = iface_at<SCH, MODE, IL>(q, opi, -1, a);
  }

  bool bad = false;
  const double2* xrow_h = a.xpsi + hcol + (ptrdiff_t)jb * ntp;
  int slot = 0;
  uint32_t parity = 0;
  for (int j = jb; j < je; ++j, xrow_h += ntp) {
    const unsigned char* sl = ring + (size_t)slot * SB;
    const int rn = j + 1 + R;
    const bool synth = (rn >= n) && a.phys_hi;
    // theta halo of this row (4 lanes, L1/L2 hits)
    double2 h = make_double2(0.0, 0.0);
    if (has_h) {
      h = ld2(xrow_h);
      if (hflip) h = neg2(h);
    }
    mbar_wait(bar0 + slot * 8, parity);
    const double2 bl = reinterpret_cast<const double2*>(sl + SlotT::BL)[lane];

    // ---- phase 1: radial derivatives
    double dpsR, dpsI, dpiR, dpiI;
    if (SCH != FD6KO) {
      double r[SW], q[SW];
#pragma unroll
      for (int m = 0; m < SW; ++m) { r[m] = wps[m].x; q[m] = wps[m].y; }
      // Psi rows: right-biased everywhere (b <= 0; evolve.cpp:103-104)
      const double cR = iface_at<SCH, MODE, SL>(r, true, 0, a);
      const double cI = iface_at<SCH, MODE, SL>(q, true, 0, a);
      dpsR = (cR - fpsR) * a.iscale; fpsR = cR;
      dpsI = (cI - fpsI) * a.iscale; fpsI = cI;
      // pi rows: minus where lam < 0 (split_k rule, evolve.cpp:19-30, 105-110)
      const bool o = bl.y < 0.0;
      double x[PW], y[PW];
#pragma unroll
      for (int m = 0; m < PW; ++m) { x[m] = wpi[m].x; y[m] = wpi[m].y; }
      if (o != opi) {
        // start of a sub-row: fresh F(j - 1/2) in the new orientation
        if (!o && SCH == WENO5) {
          // plus at j - 1/2 needs row j - 3, outside the window
          double2 u3 = row_or_ghost(xpi, j - 3, ntp, a.phys_lo);
          double xx[PW + 1], yy[PW + 1];
          xx[0] = u3.x; yy[0] = u3.y;
#pragma unroll
          for (int m = 0; m < PW; ++m) { xx[m + 1] = x[m]; yy[m + 1] = y[m]; }
          fpiR = iface_at<SCH, MODE, PL + 1>(xx, false, -1, a);
          fpiI = iface_at<SCH, MODE, PL + 1>(yy, false, -1, a);
        } else {
          fpiR = iface_at<SCH, MODE, PL>(x, o, -1, a);
          fpiI = iface_at<SCH, MODE, PL>(y, o, -1, a);
        }
        opi = o;
      }
      double pR, pI;
      if (__all_sync(kFull, !o)) {
        pR = iface_at<SCH, MODE, PL>(x, false, 0, a);
        pI = iface_at<SCH, MODE, PL>(y, false, 0, a);
      } else {
        pR = iface_at<SCH, MODE, PL>(x, o, 0, a);
        pI = iface_at<SCH, MODE, PL>(y, o, 0, a);
      }
      dpiR = (pR - fpiR) * a.iscale; fpiR = pR;
      dpiI = (pI - fpiI) * a.iscale; fpiI = pI;
    } else {
      // FD6 (spatial.hpp:178-182): centred, no upwinding, all four rows
      auto fd6 = [&](double m3, double m2, double m1, double p1, double p2, double p3) {
        return fma(45.0, p1 - m1, fma(-9.0, p2 - m2, p3 - m3)) * a.iscale;
      };
      constexpr int C = SL;
      dpsR = fd6(wps[C - 3].x, wps[C - 2].x, wps[C - 1].x, wps[C + 1].x, wps[C + 2].x, wps[C + 3].x);
      dpsI = fd6(wps[C - 3].y, wps[C - 2].y, wps[C - 1].y, wps[C + 1].y, wps[C + 2].y, wps[C + 3].y);
      dpiR = fd6(wpi[C - 3].x, wpi[C - 2].x, wpi[C - 1].x, wpi[C + 1].x, wpi[C + 2].x, wpi[C + 3].x);
      dpiI = fd6(wpi[C - 3].y, wpi[C - 2].y, wpi[C - 1].y, wpi[C + 1].y, wpi[C + 2].y, wpi[C + 3].y);
    }

    // ---- phase 2: (d_thth + cot d_th) Psi (spatial.hpp:208-222)
    const double2 ps = wps[SL];
    double2 wv = ps;   // value this lane publishes to its theta neighbours
    if (pole_chunk) {  // warp-uniform
      double2 img = make_double2(__shfl_sync(kFull, ps.x, wsrc & 31),
                                 __shfl_sync(kFull, ps.y, wsrc & 31));
      if (!active) wv = wflip ? neg2(img) : img;
    }
    const double2 su2 = shfl_up2(wv, 2), su1 = shfl_up2(wv, 1);
    const double2 sd1 = shfl_dn2(wv, 1), sd2 = shfl_dn2(wv, 2);
    const double2 hd1 = shfl_dn2(h, 1), hu1 = shfl_up2(h, 1);
    const double2 m2 = lane >= 2 ? su2 : h;
    const double2 m1 = lane >= 1 ? su1 : hd1;
    const double2 p1 = lane <= 30 ? sd1 : hu1;
    const double2 p2 = lane <= 29 ? sd2 : h;
    const double d1R = fma(8.0, p1.x - m1.x, m2.x - p2.x) * a.inv1;
    const double d1I = fma(8.0, p1.y - m1.y, m2.y - p2.y) * a.inv1;
    const double d2R = fma(-30.0, ps.x, fma(16.0, m1.x + p1.x, -(m2.x + p2.x))) * a.inv2;
    const double d2I = fma(-30.0, ps.y, fma(16.0, m1.y + p1.y, -(m2.y + p2.y))) * a.inv2;
    const double angR = fma(cot, d1R, d2R);
    const double angI = fma(cot, d1I, d2I);

    // ---- phase 3: pointwise assembly (evolve.cpp:149-167)
    const double2 cw = reinterpret_cast<const double2*>(sl + SlotT::CW)[lane];
    const double2 cbt = reinterpret_cast<const double2*>(sl + SlotT::CBT)[lane];
    const double2 ccf = reinterpret_cast<const double2*>(sl + SlotT::CCF)[lane];
    const double ath = reinterpret_cast<const double*>(sl + SlotT::ATH)[lane];
    const double2 pv = wpi[PL];
    const double b = bl.x, lam = bl.y;
    double f0 = fma(-b, dpsR, pv.x);
    double f1 = fma(-b, dpsI, pv.y);
    double f2 = fma(ath, angR, fma(-ccf.y, ps.y, fma(ccf.x, ps.x, fma(-cbt.y, pv.y,
                fma(cbt.x, pv.x, fma(-cw.y, dpsI, fma(cw.x, dpsR, -lam * dpiR)))))));
    double f3 = fma(ath, angI, fma(ccf.y, ps.x, fma(ccf.x, ps.y, fma(cbt.y, pv.x,
                fma(cbt.x, pv.y, fma(cw.y, dpsR, fma(cw.x, dpsI, -lam * dpiI)))))));
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
      f2 -= ko8(wpi[0].x, wpi[1].x, wpi[2].x, wpi[3].x, wpi[4].x, wpi[5].x, wpi[6].x, wpi[7].x, wpi[8].x);
      f3 -= ko8(wpi[0].y, wpi[1].y, wpi[2].y, wpi[3].y, wpi[4].y, wpi[5].y, wpi[6].y, wpi[7].y, wpi[8].y);
    }

    // ---- RK epilogue (timestep.hpp:61-70, 84-108), reference evaluation order
    double2 ops, opv;
    if (EPI == EPI_RHS) {
      ops = make_double2(f0, f1); opv = make_double2(f2, f3);
    } else if (EPI == EPI_AXPY) {
      ops = make_double2(ps.x + a.cg * f0, ps.y + a.cg * f1);
      opv = make_double2(pv.x + a.cg * f2, pv.y + a.cg * f3);
    } else {
      const double2 aps = reinterpret_cast<const double2*>(sl + SlotT::APS)[lane];
      const double2 api = reinterpret_cast<const double2*>(sl + SlotT::API)[lane];
      if (EPI == EPI_RK3) {
        ops = make_double2(a.ca * aps.x + a.cb * (ps.x + a.cg * f0),
                           a.ca * aps.y + a.cb * (ps.y + a.cg * f1));
        opv = make_double2(a.ca * api.x + a.cb * (pv.x + a.cg * f2),
                           a.ca * api.y + a.cb * (pv.y + a.cg * f3));
      } else if (EPI == EPI_RK104_5) {
        ops = make_double2(a.ca * aps.x + a.cb * ps.x + a.cg * f0,
                           a.ca * aps.y + a.cb * ps.y + a.cg * f1);
        opv = make_double2(a.ca * api.x + a.cb * pv.x + a.cg * f2,
                           a.ca * api.y + a.cb * pv.y + a.cg * f3);
      } else {
        const double2 bps = reinterpret_cast<const double2*>(sl + SlotT::BPS)[lane];
        const double2 bpi = reinterpret_cast<const double2*>(sl + SlotT::BPI)[lane];
        const double2 gps = reinterpret_cast<const double2*>(sl + SlotT::GPS)[lane];
        const double2 gpi = reinterpret_cast<const double2*>(sl + SlotT::GPI)[lane];
        ops = make_double2(
            a.ca * aps.x + a.cb * bps.x + a.cc * ps.x + a.cg * (a.cd * gps.x + a.ce * f0),
            a.ca * aps.y + a.cb * bps.y + a.cc * ps.y + a.cg * (a.cd * gps.y + a.ce * f1));
        opv = make_double2(
            a.ca * api.x + a.cb * bpi.x + a.cc * pv.x + a.cg * (a.cd * gpi.x + a.ce * f2),
            a.ca * api.y + a.cb * bpi.y + a.cc * pv.y + a.cg * (a.cd * gpi.y + a.ce * f3));
      }
    }
    if (active) {
      const ptrdiff_t o = (ptrdiff_t)j * ntp + k;
      a.opsi[o] = ops;
      a.opi[o] = opv;
      if (EPI == EPI_RK104_5) {
        a.fpsi[o] = make_double2(f0, f1);
        a.fpi[o] = make_double2(f2, f3);
      }
      if (a.check) {
        // state_admissible (evolve.cpp:217-235): NaN or |u| > 1e30
        bad |= !(fabs(ops.x) <= 1e30) || !(fabs(ops.y) <= 1e30) || !(fabs(opv.x) <= 1e30) ||
               !(fabs(opv.y) <= 1e30);
      }
    }

    // ---- slide the windows
#pragma unroll
    for (int m = 0; m < SW - 1; ++m) wps[m] = wps[m + 1];
#pragma unroll
    for (int m = 0; m < PW - 1; ++m) wpi[m] = wpi[m + 1];
    if (synth) {
      wps[SW - 1] = cubic(wps[SW - 2], wps[SW - 3], wps[SW - 4], wps[SW - 5]);
      wpi[PW - 1] = cubic(wpi[PW - 2], wpi[PW - 3], wpi[PW - 4], wpi[PW - 5]);
    } else {
      wps[SW - 1] = reinterpret_cast<const double2*>(sl + SlotT::XPS)[lane];
      wpi[PW - 1] = reinterpret_cast<const double2*>(sl + SlotT::XPI)[lane];
    }
    // ---- release the slot and refill it S rows ahead
    __syncwarp();
    if (lane == 0 && j + S < je) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      issue(slot, j + S);
    }
    if (++slot == S) { slot = 0; parity ^= 1u; }
  }
  if (a.check && __any_sync(kFull, bad) && lane == 0) {
    atomicExch(a.flag + 1, (unsigned long long)a.step);
    atomicOr(a.flag, 1ull);
  }
}

// ---------------------------------------------------------------------------
// Layout conversion between the reference StateVec (FieldLayout, rho fastest,
// DD {hi, lo} pairs or plain doubles) and the device planes: 32x32 tiles
// through shared memory so both sides stay coalesced.
// dir 0: host layout -> device planes (interior only); dir 1: device -> host
// layout interior (ghosts are filled on the host).
__global__ void relayout_kernel(const double* __restrict__ src, double* __restrict__ dst,
                                double2* psi, double2* pi, int n, int nt, int ntp,
                                int stride, int dir);

// Observer reduction (diagnostics.cpp:145-160, diagnostics.hpp:47-50,
// diagnostics.cpp:257-283 as a precomputed linear functional): one block.
__global__ void observe_kernel(const double2* psi, int ntp, int j0, const double* hw,
                               int kobs, int jobs, int jscri, const double* pw, int nt,
                               double* out);

}  // namespace hwg
