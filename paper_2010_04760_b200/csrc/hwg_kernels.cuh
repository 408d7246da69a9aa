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

// reference cubic continuation p[-t] = 4p[-t+1] - 6p[-t+2] + 4p[-t+3] - p[-t+4]
// (evolve.cpp:48-50), same evaluation order
__device__ __forceinline__ double cubic1(double a, double b, double c, double d) {
  return 4.0 * a - 6.0 * b + 4.0 * c - d;
}
__device__ __forceinline__ double2 cubic(double2 a, double2 b, double2 c, double2 d) {
  return make_double2(cubic1(a.x, b.x, c.x, d.x), cubic1(a.y, b.y, c.y, d.y));
}

// ---------------------------------------------------------------------------
// WENO5-JS interface value (spatial.hpp:29-92) on the oriented window
// f0..f4, returned WITHOUT the 1/6 factor (folded into iscale).
//
// fp64 weights: alpha_k = d_k/(eps + IS_k)^2 normalised; with the indicators
// scaled by 4 (IS' = 13/3 t^2 + s^2, eps' = 4 eps) the weights are
// w_k = d_k prod_{i!=k} e_i^2 / sum(...), so one reciprocal replaces the
// reference's five divisions.
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
  return num * __drcp_rn((n0 + n1) + n2);
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
    float a0 = 0.1f * __frcp_rn(e0 * e0);
    float a1 = 0.6f * __frcp_rn(e1 * e1);
    float a2 = 0.3f * __frcp_rn(e2 * e2);
    float inv = __frcp_rn((a0 + a1) + a2);
    w0 = a0 * inv; w1 = a1 * inv; w2 = a2 * inv;
  }
  const double W0 = (double)w0, W1 = (double)w1, W2 = (double)w2;
  double c0 = fma(11.0, f2, fma(-7.0, f1, 2.0 * f0));
  double c1 = fma(2.0, f3, fma(5.0, f2, -f1));
  double c2 = fma(5.0, f3, fma(2.0, f2, -f4));
  double num = fma(W2, c2, fma(W1, c1, W0 * c0));
  return num * __drcp_rn((W0 + W1) + W2);
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
    float x0 = (1.0f / 3.0f) * __frcp_rn(e0 * e0);
    float x1 = (2.0f / 3.0f) * __frcp_rn(e1 * e1);
    float inv = __frcp_rn(x0 + x1);
    n0 = (double)(x0 * inv);
    n1 = (double)(x1 * inv);
  }
  double q0 = fma(3.0, f1, -f0);
  double q1 = f1 + f2;
  return fma(n1, q1, n0 * q0) * __drcp_rn(n0 + n1);
}

// ---------------------------------------------------------------------------
// theta neighbour Psi(j, k + d) of every lane: warp shuffle when the
// (parity-reflected) source column lies in this warp's chunk, a direct load
// for the few edge lanes whose source lies in the neighbouring chunk.
__device__ __forceinline__ double2 theta_nb(double2 v, int d, int k, int k0, int nt, bool active,
                                            int negpar, const double2* row) {
  int kk = k + d;
  bool flip = false;
  if (kk < 0) { kk = -1 - kk; flip = negpar; }
  else if (kk >= nt) { kk = 2 * nt - 1 - kk; flip = negpar; }
  const int src = kk - k0;
  const bool in = (src >= 0) && (src < 32);
  const int sl = in ? src : (threadIdx.x & 31);
  double2 r;
  r.x = __shfl_sync(kFull, v.x, sl);
  r.y = __shfl_sync(kFull, v.y, sl);
  if (!in && active) r = ld2(row + kk);
  return flip ? neg2(r) : r;
}

// ---------------------------------------------------------------------------
template <int SCH>
struct Win {
  // window rows j - L .. j + R around the point being updated
  static constexpr int L = (SCH == FD6KO) ? 4 : (SCH == WENO5 ? 3 : 2);
  static constexpr int R = L;
  static constexpr int W = L + R + 1;
};

template <int SCH, int MODE, int EPI>
__global__ void __launch_bounds__(kWarpsPerBlock * 32)
stage_kernel(const StageArgs a) {
  if (a.flag != nullptr && *(volatile unsigned long long*)a.flag != 0ull) return;  // frozen
  constexpr int L = Win<SCH>::L, W = Win<SCH>::W, C = L;
  const int lane = threadIdx.x & 31;
  const int gw = blockIdx.x * kWarpsPerBlock + (threadIdx.x >> 5);
  const int chunk = gw % a.nchunks;
  const int range = gw / a.nchunks;
  if (range >= a.nranges) return;                       // whole warp
  const int jb = (int)((long long)range * a.n / a.nranges);
  const int je = (int)((long long)(range + 1) * a.n / a.nranges);
  const int k0 = chunk << 5;
  const int k = k0 + lane;
  const bool active = k < a.nt;
  const int kc = active ? k : a.nt - 1;
  const int ntp = a.ntp, n = a.n;

  const double2* xps = a.xpsi + kc;
  const double2* xpi = a.xpi + kc;

  // ---- window initialisation: rows jb - L .. jb + R
  double2 wps[W], wpi[W];
  if (a.phys_lo && jb == 0) {
    double2 qs[L + 4], qp[L + 4];
#pragma unroll
    for (int m = 0; m < 4; ++m) {
      qs[L + m] = ld2(xps + (size_t)m * ntp);
      qp[L + m] = ld2(xpi + (size_t)m * ntp);
    }
#pragma unroll
    for (int t = 1; t <= L; ++t) {
      qs[L - t] = cubic(qs[L - t + 1], qs[L - t + 2], qs[L - t + 3], qs[L - t + 4]);
      qp[L - t] = cubic(qp[L - t + 1], qp[L - t + 2], qp[L - t + 3], qp[L - t + 4]);
    }
#pragma unroll
    for (int m = 0; m < W; ++m) {
      if (m < L + 4) { wps[m] = qs[m]; wpi[m] = qp[m]; }
      else {
        wps[m] = ld2(xps + (size_t)(m - L) * ntp);
        wpi[m] = ld2(xpi + (size_t)(m - L) * ntp);
      }
    }
  } else {
#pragma unroll
    for (int m = 0; m < W; ++m) {
      const int r = jb - L + m;
      if (r >= n && a.phys_hi) {
        wps[m] = cubic(wps[m - 1], wps[m - 2], wps[m - 3], wps[m - 4]);
        wpi[m] = cubic(wpi[m - 1], wpi[m - 2], wpi[m - 3], wpi[m - 4]);
      } else {
        wps[m] = ld2(xps + (ptrdiff_t)r * ntp);
        wpi[m] = ld2(xpi + (ptrdiff_t)r * ntp);
      }
    }
  }

  // pointwise data of the current row (software pipelined one row ahead)
  const size_t pk = kc;
  auto ldpt = [&](int j, double2& bl, double2& w, double2& bt, double2& cf, double& ath,
                  double2& aps, double2& api, double2& bps, double2& bpi, double2& gps,
                  double2& gpi) {
    const size_t o = (size_t)j * ntp + pk;
    bl = ld2(a.cbl + o); w = ld2(a.cw + o); bt = ld2(a.cbt + o); cf = ld2(a.ccf + o);
    ath = __ldg(a.cath + o);
    if (EPI == EPI_RK3 || EPI == EPI_RK104_5 || EPI == EPI_RK104_10) {
      aps = a.apsi[o]; api = a.api[o];
    }
    if (EPI == EPI_RK104_10) {
      bps = a.bpsi[o]; bpi = a.bpi[o]; gps = a.gpsi[o]; gpi = a.gpi[o];
    }
  };
  double2 bl, cw, cbt, ccf, aps, api, bps, bpi, gps, gpi;
  double ath;
  ldpt(jb, bl, cw, cbt, ccf, ath, aps, api, bps, bpi, gps, gpi);
  const double cot = __ldg(a.cot + kc);

  // carried interface values F(j - 1/2)
  double fpsR = 0.0, fpsI = 0.0, fpiR = 0.0, fpiI = 0.0;
  int opi = -1;  // orientation of the carried pi interfaces (1 = minus)
  if (SCH == WENO5) {
    fpsR = weno5<MODE>(wps[C + 2].x, wps[C + 1].x, wps[C].x, wps[C - 1].x, wps[C - 2].x, a);
    fpsI = weno5<MODE>(wps[C + 2].y, wps[C + 1].y, wps[C].y, wps[C - 1].y, wps[C - 2].y, a);
  } else if (SCH == WENO3) {
    fpsR = weno3<MODE>(wps[C + 1].x, wps[C].x, wps[C - 1].x, a);
    fpsI = weno3<MODE>(wps[C + 1].y, wps[C].y, wps[C - 1].y, a);
  }

  bool bad = false;
  for (int j = jb; j < je; ++j) {
    // ---- prefetch next row (state row j + 1 + R and pointwise row j + 1)
    const bool more = j + 1 < je;
    const int rn = j + 1 + Win<SCH>::R;
    const bool synth = (rn >= n) && a.phys_hi;
    double2 nps = make_double2(0.0, 0.0), npi = nps;
    double2 nbl = nps, ncw = nps, ncbt = nps, nccf = nps, naps = nps, napi = nps, nbps = nps,
            nbpi = nps, ngps = nps, ngpi = nps;
    double nath = 0.0;
    if (more) {
      if (!synth) {
        nps = ld2(xps + (ptrdiff_t)rn * ntp);
        npi = ld2(xpi + (ptrdiff_t)rn * ntp);
      }
      ldpt(j + 1, nbl, ncw, ncbt, nccf, nath, naps, napi, nbps, nbpi, ngps, ngpi);
    }

    // ---- phase 1: radial derivatives
    double dpsR, dpsI, dpiR, dpiI;
    if (SCH == WENO5) {
      double cR = weno5<MODE>(wps[C + 3].x, wps[C + 2].x, wps[C + 1].x, wps[C].x, wps[C - 1].x, a);
      double cI = weno5<MODE>(wps[C + 3].y, wps[C + 2].y, wps[C + 1].y, wps[C].y, wps[C - 1].y, a);
      dpsR = (cR - fpsR) * a.iscale; fpsR = cR;
      dpsI = (cI - fpsI) * a.iscale; fpsI = cI;
      const int o = bl.y < 0.0;   // split_k rule: minus where lam < 0 (evolve.cpp:19-30)
      if (o != opi) {             // start of a (sub-)row: fresh F(j - 1/2)
        double2 f0 = o ? wpi[C + 2] : wpi[C - 3], f1 = o ? wpi[C + 1] : wpi[C - 2],
                f2 = o ? wpi[C] : wpi[C - 1], f3 = o ? wpi[C - 1] : wpi[C],
                f4 = o ? wpi[C - 2] : wpi[C + 1];
        fpiR = weno5<MODE>(f0.x, f1.x, f2.x, f3.x, f4.x, a);
        fpiI = weno5<MODE>(f0.y, f1.y, f2.y, f3.y, f4.y, a);
        opi = o;
      }
      double2 f0 = o ? wpi[C + 3] : wpi[C - 2], f1 = o ? wpi[C + 2] : wpi[C - 1],
              f2 = o ? wpi[C + 1] : wpi[C], f3 = o ? wpi[C] : wpi[C + 1],
              f4 = o ? wpi[C - 1] : wpi[C + 2];
      double pR = weno5<MODE>(f0.x, f1.x, f2.x, f3.x, f4.x, a);
      double pI = weno5<MODE>(f0.y, f1.y, f2.y, f3.y, f4.y, a);
      dpiR = (pR - fpiR) * a.iscale; fpiR = pR;
      dpiI = (pI - fpiI) * a.iscale; fpiI = pI;
    } else if (SCH == WENO3) {
      double cR = weno3<MODE>(wps[C + 2].x, wps[C + 1].x, wps[C].x, a);
      double cI = weno3<MODE>(wps[C + 2].y, wps[C + 1].y, wps[C].y, a);
      dpsR = (cR - fpsR) * a.iscale; fpsR = cR;
      dpsI = (cI - fpsI) * a.iscale; fpsI = cI;
      const int o = bl.y < 0.0;
      if (o != opi) {
        double2 f0 = o ? wpi[C + 1] : wpi[C - 2], f1 = o ? wpi[C] : wpi[C - 1],
                f2 = o ? wpi[C - 1] : wpi[C];
        fpiR = weno3<MODE>(f0.x, f1.x, f2.x, a);
        fpiI = weno3<MODE>(f0.y, f1.y, f2.y, a);
        opi = o;
      }
      double2 f0 = o ? wpi[C + 2] : wpi[C - 1], f1 = o ? wpi[C + 1] : wpi[C],
              f2 = o ? wpi[C] : wpi[C + 1];
      double pR = weno3<MODE>(f0.x, f1.x, f2.x, a);
      double pI = weno3<MODE>(f0.y, f1.y, f2.y, a);
      dpiR = (pR - fpiR) * a.iscale; fpiR = pR;
      dpiI = (pI - fpiI) * a.iscale; fpiI = pI;
    } else {
      // FD6 (spatial.hpp:178-182): centred, no upwinding, all four rows
      auto fd6 = [&](double m3, double m2, double m1, double p1, double p2, double p3) {
        return fma(45.0, p1 - m1, fma(-9.0, p2 - m2, p3 - m3)) * a.iscale;
      };
      dpsR = fd6(wps[C - 3].x, wps[C - 2].x, wps[C - 1].x, wps[C + 1].x, wps[C + 2].x, wps[C + 3].x);
      dpsI = fd6(wps[C - 3].y, wps[C - 2].y, wps[C - 1].y, wps[C + 1].y, wps[C + 2].y, wps[C + 3].y);
      dpiR = fd6(wpi[C - 3].x, wpi[C - 2].x, wpi[C - 1].x, wpi[C + 1].x, wpi[C + 2].x, wpi[C + 3].x);
      dpiI = fd6(wpi[C - 3].y, wpi[C - 2].y, wpi[C - 1].y, wpi[C + 1].y, wpi[C + 2].y, wpi[C + 3].y);
    }

    // ---- phase 2: (d_thth + cot d_th) Psi (spatial.hpp:208-222)
    const double2 ps = wps[C];
    const double2* xrow = a.xpsi + (ptrdiff_t)j * ntp;
    const double2 m2 = theta_nb(ps, -2, k, k0, a.nt, active, a.negpar, xrow);
    const double2 m1 = theta_nb(ps, -1, k, k0, a.nt, active, a.negpar, xrow);
    const double2 p1 = theta_nb(ps, 1, k, k0, a.nt, active, a.negpar, xrow);
    const double2 p2 = theta_nb(ps, 2, k, k0, a.nt, active, a.negpar, xrow);
    const double d1R = fma(8.0, p1.x - m1.x, m2.x - p2.x) * a.inv1;
    const double d1I = fma(8.0, p1.y - m1.y, m2.y - p2.y) * a.inv1;
    const double d2R = fma(-30.0, ps.x, fma(16.0, m1.x + p1.x, -(m2.x + p2.x))) * a.inv2;
    const double d2I = fma(-30.0, ps.y, fma(16.0, m1.y + p1.y, -(m2.y + p2.y))) * a.inv2;
    const double angR = fma(cot, d1R, d2R);
    const double angI = fma(cot, d1I, d2I);

    // ---- phase 3: pointwise assembly (evolve.cpp:149-167)
    const double2 pv = wpi[C];
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
    } else if (EPI == EPI_RK3) {
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
      ops = make_double2(
          a.ca * aps.x + a.cb * bps.x + a.cc * ps.x + a.cg * (a.cd * gps.x + a.ce * f0),
          a.ca * aps.y + a.cb * bps.y + a.cc * ps.y + a.cg * (a.cd * gps.y + a.ce * f1));
      opv = make_double2(
          a.ca * api.x + a.cb * bpi.x + a.cc * pv.x + a.cg * (a.cd * gpi.x + a.ce * f2),
          a.ca * api.y + a.cb * bpi.y + a.cc * pv.y + a.cg * (a.cd * gpi.y + a.ce * f3));
    }
    if (active) {
      const size_t o = (size_t)j * ntp + k;
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

    // ---- slide the window
#pragma unroll
    for (int m = 0; m < W - 1; ++m) { wps[m] = wps[m + 1]; wpi[m] = wpi[m + 1]; }
    if (synth) {
      wps[W - 1] = cubic(wps[W - 2], wps[W - 3], wps[W - 4], wps[W - 5]);
      wpi[W - 1] = cubic(wpi[W - 2], wpi[W - 3], wpi[W - 4], wpi[W - 5]);
    } else {
      wps[W - 1] = nps; wpi[W - 1] = npi;
    }
    bl = nbl; cw = ncw; cbt = ncbt; ccf = nccf; ath = nath;
    aps = naps; api = napi; bps = nbps; bpi = nbpi; gps = ngps; gpi = ngpi;
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
