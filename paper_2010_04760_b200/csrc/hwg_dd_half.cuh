// Double-double stage kernel, lane = (theta column, component) form.
//
// The same arithmetic as hwg_dd.cuh's first form (the reference's DDReal
// operations in its evaluation order, bitwise), mapped differently: a warp
// owns HALF a 32-column chunk and each lane one COMPONENT (real or imaginary
// part) of one column: lane l -> column k0 + l/2, component l & 1.  A lane's
// register windows then hold one component of Psi and pi instead of both
// (half the live state), so the kernel fits 168 registers and 12 warps per SM
// (3 per scheduler) instead of 255 registers and 8 — the FP64 pipe sees a
// third more independent double-double chains (ncu: the first form spends
// ~37 % of its cycles waiting on fixed-latency dependencies at 2 warps per
// scheduler).  The complex products of the assembly
// (evolve.cpp:149-167) take their partner component with one shuffle
// (lanes l and l ^ 1 hold the two parts of a column), every other operation
// is per component, so each lane executes the reference's operation sequence
// for its component exactly as the first form does.
//
// Data layout in HBM is unchanged (hwg_dd.cuh): a lane reads the doubles
// q*64 + h*32 + l of a state block (q = Psi.hi, pi.hi, Psi.lo, pi.lo; h =
// the half) — 256 contiguous bytes per warp and part.  The bulk-copy ring
// brings the half's 16 columns of the coefficient and state blocks.
#pragma once

#include "hwg_dd.cuh"

namespace hwg {

constexpr int kDDWarpsPerChunk = 2;

// state-block half in shared memory: [Psi.hi | pi.hi | Psi.lo | pi.lo], 16 double2 each
__device__ __forceinline__ dd sm_half(const double* blk, int part, int lane) {
  return {blk[part * 32 + lane], blk[64 + part * 32 + lane]};
}
// the same doubles of a global state block (row, chunk) for half h
__device__ __forceinline__ dd ld_half(const double2* blk, int part, int h, int lane) {
  const double* p = reinterpret_cast<const double*>(blk) + h * 32;
  return {__ldg(p + part * 64 + lane), __ldg(p + 128 + part * 64 + lane)};
}
// component `comp` of column `col` (any chunk) of a global state row
__device__ __forceinline__ dd ld_col(const double2* row0, int col, int part, int comp) {
  const double* p = reinterpret_cast<const double*>(row0 + (col >> 5) * kStateBlkDD);
  const int i = (part * 32 + (col & 31)) * 2 + comp;
  return {__ldg(p + i), __ldg(p + 128 + i)};
}

template <int EPI>
struct SlotDH {
  static constexpr int COEF = 0;            // [hi: 4 x 16 double2 + 16 ath | lo: same] 2304 B
  static constexpr int CPART = 72;          // double2 per limb part
  static constexpr int XN = 2 * CPART * 16; // next stencil row, 1024 B
  static constexpr int A = XN + 1024;
  static constexpr bool HAS_A = EPI >= EPI_RK3;
  static constexpr bool HAS_BG = EPI == EPI_RK104_10;
  static constexpr int B = A + (HAS_A ? 1024 : 0);
  static constexpr int G = B + 1024;
  static constexpr int BYTES = B + (HAS_BG ? 2048 : 0);
  static constexpr int S = 2;
};
template <int EPI>
__host__ __device__ constexpr size_t stage_theta_offset_dh(int wpb) {
  return ((size_t)wpb * SlotDH<EPI>::S * (SlotDH<EPI>::BYTES + 8) + 15) & ~(size_t)15;
}
// per warp: the theta-extended Psi row E[(i, comp)], i < 20 columns k0-2 .. k0+17
template <int EPI>
constexpr size_t stage_smem_bytes_dd(int wpb = kWarpsPerBlock) {
  return stage_theta_offset_dh<EPI>(wpb) + (size_t)wpb * 40 * sizeof(dd);
}

template <int SCH, int MODE, int C, int N>
__device__ __forceinline__ dd iface_h(const dd (&w)[N], bool minus, int shift, const StageArgsDD& A) {
  const int c = C + shift;
  if (SCH == WENO5)
    return minus ? iface_one_call<SCH, MODE>(w[c + 3], w[c + 2], w[c + 1], w[c], w[c - 1], A.kdev, A.eps_hi)
                 : iface_one_call<SCH, MODE>(w[c - 2], w[c - 1], w[c], w[c + 1], w[c + 2], A.kdev, A.eps_hi);
  return minus ? iface_one_call<SCH, MODE>(w[c + 2], w[c + 1], w[c], w[c], w[c], A.kdev, A.eps_hi)
               : iface_one_call<SCH, MODE>(w[c - 1], w[c], w[c + 1], w[c], w[c], A.kdev, A.eps_hi);
}

static __device__ __noinline__ dd row_or_ghost_h(const double2* xblk, int h, int lane, int r,
                                                  ptrdiff_t rs, int phys_lo, const DDConsts& K) {
  if (r >= 0 || !phys_lo) return ld_half(xblk + r * rs, 1, h, lane);
  dd g[8];
  for (int m = 0; m < 4; ++m) g[4 + m] = ld_half(xblk + m * rs, 1, h, lane);
  for (int t = 1; t <= -r; ++t) g[4 - t] = cubic_dd(g[4 - t + 1], g[4 - t + 2], g[4 - t + 3], g[4 - t + 4], K);
  return g[4 + r];
}

#ifndef HWG_DD_MINB
#define HWG_DD_MINB 3
#endif
template <int SCH, int MODE, int EPI, bool INL>
__global__ void __launch_bounds__(kWarpsPerBlock * 32, HWG_DD_MINB)
stage_kernel_dd(const StageArgsDD A) {
  if (A.flag != nullptr && *(volatile unsigned long long*)A.flag != 0ull) return;
  if (A.bump && blockIdx.x == 0 && threadIdx.x == 0) A.flag[2] += 1ull;  // step counter
  using Wn = Win<SCH>;
  using SlotT = SlotDH<EPI>;
  constexpr int SL = Wn::SL, PL = Wn::PL, R = Wn::R, SW = Wn::SW, PW = Wn::PW;
  constexpr int IL = Wn::IL, IW = Wn::IW, S = SlotT::S, SB = SlotT::BYTES;
  constexpr bool CHECK = EPI == EPI_RK3C || EPI == EPI_RK104_10;
  const DDConsts& K = A.k;
  extern __shared__ __align__(128) unsigned char smem[];
  const int lane = threadIdx.x & 31;
  const int wib = threadIdx.x >> 5;
  const int wpb = blockDim.x >> 5;
  const int gw = blockIdx.x * wpb + wib;
  const int nhalf = 2 * A.nchunks;
  const int hidx = gw % nhalf;
  const int range = gw / nhalf;
  if (range >= A.nranges) return;
  const int chunk = hidx >> 1, h = hidx & 1;
  const int jb = (int)((long long)range * A.n / A.nranges);
  const int je = (int)((long long)(range + 1) * A.n / A.nranges);
  const int cc = lane >> 1;            // column within the half
  const int comp = lane & 1;           // 0 real, 1 imaginary part
  const int k0 = chunk * 32 + h * 16;  // first column of the half
  const int k = k0 + cc;
  const int nt = A.nt, n = A.n;
  const bool active = k < nt;
  const ptrdiff_t rs = (ptrdiff_t)A.nchunks * kStateBlkDD;
  const ptrdiff_t crs = (ptrdiff_t)A.nchunks * kCoefBlkDD;
  // theta halo columns k0-2, k0-1 (lanes 0-3) and k0+16, k0+17 (lanes 28-31)
  const bool has_h = lane < 4 || lane >= 28;
  bool hflip;
  const int hcol = reflect_col(lane < 4 ? k0 - 2 + cc : k0 + 16 + (cc - 14), nt, hflip, A.negpar);
  const bool pole_half = k0 + 16 > nt;
  bool wflip;
  const int wcol = reflect_col(k, nt, wflip, A.negpar);
  const int wsrc = wcol - k0;          // image column's index in this half (if 0..15)

  unsigned char* ring = smem + (size_t)wib * S * SB;
  const uint32_t bar0 = smem_u32(smem + (size_t)wpb * S * SB) + wib * S * 8;
  const double2* xblk = A.x + chunk * kStateBlkDD;
  const double2* cblk = A.coef + chunk * kCoefBlkDD;
  auto issue = [&](int s, int j) {
    const uint32_t bar = bar0 + s * 8;
    const uint32_t dst = smem_u32(ring + (size_t)s * SB);
    const int rn = j + 1 + R;
    const bool st = (j + 1 < je) && !(rn >= n && A.phys_hi);
    mbar_expect_tx(bar, SlotT::BYTES - (st ? 0 : 1024));
    const double2* cs = cblk + j * crs;
#pragma unroll
    for (int p = 0; p < 2; ++p) {  // hi, lo limb blocks
#pragma unroll
      for (int m = 0; m < 4; ++m)
        bulk_g2s(dst + (p * SlotT::CPART + m * 16) * 16, cs + p * kCoefBlk + m * 32 + h * 16, 256, bar);
      bulk_g2s(dst + (p * SlotT::CPART + 64) * 16,
               reinterpret_cast<const double*>(cs + p * kCoefBlk + kCoefAth) + h * 16, 128, bar);
    }
    const ptrdiff_t o = j * rs + chunk * kStateBlkDD + h * 16;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      if (st) bulk_g2s(dst + SlotT::XN + q * 256, xblk + rn * rs + h * 16 + q * 32, 256, bar);
      if (SlotT::HAS_A) bulk_g2s(dst + SlotT::A + q * 256, A.ua + o + q * 32, 256, bar);
      if (SlotT::HAS_BG) {
        bulk_g2s(dst + SlotT::B + q * 256, A.ub + o + q * 32, 256, bar);
        bulk_g2s(dst + SlotT::G + q * 256, A.ug + o + q * 32, 256, bar);
      }
    }
  };
  if (lane == 0) {
    for (int s = 0; s < S; ++s) mbar_init(bar0 + s * 8, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    for (int q = 0; q < S && jb + q < je; ++q) issue(q, jb + q);
  }
  __syncwarp();

  // ---- initial rows
  dd ips[Wn::IA], ipi[Wn::IA];
  if (A.phys_lo && jb < IL) {
#pragma unroll
    for (int m = 0; m < 4; ++m) {
      ips[IL + m] = ld_half(xblk + m * rs, 0, h, lane);
      ipi[IL + m] = ld_half(xblk + m * rs, 1, h, lane);
    }
#pragma unroll
    for (int t = 1; t <= IL; ++t) {
      ips[IL - t] = cubic_dd(ips[IL - t + 1], ips[IL - t + 2], ips[IL - t + 3], ips[IL - t + 4], K);
      ipi[IL - t] = cubic_dd(ipi[IL - t + 1], ipi[IL - t + 2], ipi[IL - t + 3], ipi[IL - t + 4], K);
    }
#pragma unroll
    for (int m = IL + 4; m < IW; ++m) {
      ips[m] = ld_half(xblk + (m - IL) * rs, 0, h, lane);
      ipi[m] = ld_half(xblk + (m - IL) * rs, 1, h, lane);
    }
  } else {
#pragma unroll
    for (int m = 0; m < IW; ++m) {
      const int r = jb - IL + m;
      if (r >= n && A.phys_hi) {
        ips[m] = cubic_dd(ips[m - 1], ips[m - 2], ips[m - 3], ips[m - 4], K);
        ipi[m] = cubic_dd(ipi[m - 1], ipi[m - 2], ipi[m - 3], ipi[m - 4], K);
      } else {
        ips[m] = ld_half(xblk + r * rs, 0, h, lane);
        ipi[m] = ld_half(xblk + r * rs, 1, h, lane);
      }
    }
  }
  dd wps[SW], wpi[PW];
#pragma unroll
  for (int m = 0; m < SW; ++m) wps[m] = ips[IL - SL + m];
#pragma unroll
  for (int m = 0; m < PW; ++m) wpi[m] = ipi[IL - PL + m];

  const dd cot = A.cot[k];
  dd fps = D(0.0), fpi = D(0.0);
  bool opi = __ldg(&cblk[jb * crs + h * 16 + cc].y) < 0.0;
  if (SCH != FD6KO) {
    fps = iface_h<SCH, MODE, IL>(ips, true, -1, A);
    fpi = iface_h<SCH, MODE, IL>(ipi, opi, -1, A);
  }

  bool bad = false;
  int slot = 0;
  uint32_t parity = 0;
  dd* trow = reinterpret_cast<dd*>(smem + stage_theta_offset_dh<EPI>(wpb)) + wib * 40;
  for (int j = jb; j < je; ++j) {
    const unsigned char* sl = ring + (size_t)slot * SB;
    const double2* sc = reinterpret_cast<const double2*>(sl);
    mbar_wait(bar0 + slot * 8, parity);
    auto coef = [&](int m) -> dd2 {  // member m (double2 pair) of this column's coefficients
      const double2 hi = sc[m * 16 + cc], lo = sc[SlotT::CPART + m * 16 + cc];
      return {{hi.x, lo.x}, {hi.y, lo.y}};
    };
    const dd2 bl = coef(0);  // (b, lam)
    const dd b = bl.re, lam = bl.im;

    // ---- phase 1 (evolve.cpp:88-122), this lane's component
    dd dps, dpi;
    if (SCH != FD6KO) {
#ifdef HWG_DD_PAIR
      // both interfaces of the row (Psi, always minus; pi in its orientation)
      // in one call: two independent chains for the scheduler
      const bool o = lam.hi < 0.0;  // split_ rule (evolve.cpp:22)
      if (o != opi) {
        if (!o && SCH == WENO5) {
          dd xx[PW + 1];
          xx[0] = row_or_ghost_h(xblk, h, lane, j - 3, rs, A.phys_lo, K);
#pragma unroll
          for (int m = 0; m < PW; ++m) xx[m + 1] = wpi[m];
          fpi = iface_h<SCH, MODE, PL + 1>(xx, false, -1, A);
        } else {
          fpi = iface_h<SCH, MODE, PL>(wpi, o, -1, A);
        }
        opi = o;
      }
      constexpr int cs_ = SL, cp_ = PL;
      const dd2 r = SCH == WENO5
          ? iface_two_call<SCH, MODE>(wps[cs_ + 3], wps[cs_ + 2], wps[cs_ + 1], wps[cs_], wps[cs_ - 1],
                                      o ? wpi[cp_ + 3] : wpi[cp_ - 2], o ? wpi[cp_ + 2] : wpi[cp_ - 1],
                                      o ? wpi[cp_ + 1] : wpi[cp_], o ? wpi[cp_] : wpi[cp_ + 1],
                                      o ? wpi[cp_ - 1] : wpi[cp_ + 2], A.kdev, A.eps_hi)
          : iface_two_call<SCH, MODE>(wps[cs_ + 2], wps[cs_ + 1], wps[cs_], wps[cs_], wps[cs_],
                                      o ? wpi[cp_ + 2] : wpi[cp_ - 1], o ? wpi[cp_ + 1] : wpi[cp_],
                                      o ? wpi[cp_] : wpi[cp_ + 1], wpi[cp_], wpi[cp_], A.kdev, A.eps_hi);
      dps = (r.re - fps) * K.inv_drho;
      fps = r.re;
      dpi = (r.im - fpi) * K.inv_drho;
      fpi = r.im;
#else
      const dd cs = iface_h<SCH, MODE, SL>(wps, true, 0, A);
      dps = (cs - fps) * K.inv_drho;
      fps = cs;
      const bool o = lam.hi < 0.0;  // split_ rule (evolve.cpp:22)
      if (o != opi) {
        if (!o && SCH == WENO5) {
          dd xx[PW + 1];
          xx[0] = row_or_ghost_h(xblk, h, lane, j - 3, rs, A.phys_lo, K);
#pragma unroll
          for (int m = 0; m < PW; ++m) xx[m + 1] = wpi[m];
          fpi = iface_h<SCH, MODE, PL + 1>(xx, false, -1, A);
        } else {
          fpi = iface_h<SCH, MODE, PL>(wpi, o, -1, A);
        }
        opi = o;
      }
      dd pp;
      if (__all_sync(kFull, !o)) pp = iface_h<SCH, MODE, PL>(wpi, false, 0, A);
      else pp = iface_h<SCH, MODE, PL>(wpi, o, 0, A);
      dpi = (pp - fpi) * K.inv_drho;
      fpi = pp;
#endif
    } else {
      // fd6_derivative (spatial.hpp:178-182)
      auto fd6 = [&](dd m3, dd m2, dd m1, dd p1, dd p2, dd p3) {
        return (p3 - m3 - mul_c(p2 - m2, 9.0) + mul_c(p1 - m1, 45.0)) / K.h60;
      };
      constexpr int C = SL;
      dps = fd6(wps[C - 3], wps[C - 2], wps[C - 1], wps[C + 1], wps[C + 2], wps[C + 3]);
      dpi = fd6(wpi[C - 3], wpi[C - 2], wpi[C - 1], wpi[C + 1], wpi[C + 2], wpi[C + 3]);
    }

    // ---- phase 2: theta_derivatives_column (spatial.hpp:208-222)
    const dd ps = wps[SL];
    dd wv = ps;
    if (pole_half) {  // columns past the pole hold the parity images
      dd img = {__shfl_sync(kFull, ps.hi, ((wsrc & 15) << 1) | comp),
                __shfl_sync(kFull, ps.lo, ((wsrc & 15) << 1) | comp)};
      if (!active && (wsrc < 0 || wsrc > 15)) img = ld_col(A.x + (ptrdiff_t)j * rs, wcol, 0, comp);
      if (!active) wv = wflip ? -img : img;
    }
    dd hv = D(0.0);
    if (has_h) {
      hv = ld_col(A.x + (ptrdiff_t)j * rs, hcol, 0, comp);
      if (hflip) hv = -hv;
    }
    trow[(cc + 2) * 2 + comp] = wv;
    if (lane < 4) trow[lane] = hv;             // columns k0-2, k0-1
    else if (lane >= 28) trow[lane + 8] = hv;  // columns k0+16, k0+17
    __syncwarp();
    const dd m2 = trow[cc * 2 + comp], m1 = trow[(cc + 1) * 2 + comp];
    const dd p1 = trow[(cc + 3) * 2 + comp], p2 = trow[(cc + 4) * 2 + comp];
    const dd d1 = (m2 - mul_p2(m1, 8.0) + mul_p2(p1, 8.0) - p2) * K.inv1;
    const dd d2 = (-m2 + mul_p2(m1, 16.0) - mul_c(ps, 30.0) + mul_p2(p1, 16.0) - p2) * K.inv2;
    const dd ang = d2 + cot * d1;

    // ---- phase 3 (evolve.cpp:149-167): Psi row f_c = pi_c - b dPsi_c; pi row
    // -lam dpi_c + W dPsi + BT pi + C Psi + ath ang_c, the complex products'
    // partner component (lane ^ 1) by shuffle, the real part's three
    // subtractions as additions of negated products like the reference's a - b
    const dd2 cw = coef(1), cbt = coef(2), ccf = coef(3);
    const dd ath = {reinterpret_cast<const double*>(sc + 64)[cc],
                    reinterpret_cast<const double*>(sc + SlotT::CPART + 64)[cc]};
    const dd pv = wpi[PL];
    const dd dps_p = {__shfl_xor_sync(kFull, dps.hi, 1), __shfl_xor_sync(kFull, dps.lo, 1)};
    const dd pv_p = {__shfl_xor_sync(kFull, pv.hi, 1), __shfl_xor_sync(kFull, pv.lo, 1)};
    const dd ps_p = {__shfl_xor_sync(kFull, ps.hi, 1), __shfl_xor_sync(kFull, ps.lo, 1)};
    dd fs = pv - b * dps;
    const dd x3 = cw.im * dps_p, x5 = cbt.im * pv_p, x7 = ccf.im * ps_p;
    dd fp = -lam * dpi + cw.re * dps + (comp ? x3 : -x3) + cbt.re * pv + (comp ? x5 : -x5) +
            ccf.re * ps + (comp ? x7 : -x7) + ath * ang;
    if (SCH == FD6KO) {
      // ko8_dissipation (spatial.hpp:184-191), evolve.cpp:169-176
      auto ko8 = [&](dd u4m, dd u3m, dd u2m, dd u1m, dd u0, dd u1p, dd u2p, dd u3p, dd u4p) {
        dd d8 = u4m + u4p - mul_p2(u3m + u3p, 8.0) + mul_c(u2m + u2p, 28.0) -
                mul_c(u1m + u1p, 56.0) + mul_c(u0, 70.0);
        return K.sigma * d8 / K.h256;
      };
      fs = fs - ko8(wps[0], wps[1], wps[2], wps[3], wps[4], wps[5], wps[6], wps[7], wps[8]);
      fp = fp - ko8(wpi[0], wpi[1], wpi[2], wpi[3], wpi[4], wpi[5], wpi[6], wpi[7], wpi[8]);
    }

    // ---- epilogue (timestep.hpp:61-70, 84-108)
    dd os, op;
    if (EPI == EPI_RHS) {
      os = fs;
      op = fp;
    } else if (EPI == EPI_AXPY) {
      os = ps + K.cg * fs;
      op = pv + K.cg * fp;
    } else {
      const double* sa = reinterpret_cast<const double*>(sl + SlotT::A);
      const dd as = sm_half(sa, 0, lane), ap = sm_half(sa, 1, lane);
      if (EPI == EPI_RK3 || EPI == EPI_RK3C) {
        os = K.ca * as + K.cb * (ps + K.cg * fs);
        op = K.ca * ap + K.cb * (pv + K.cg * fp);
      } else if (EPI == EPI_RK104_5) {
        os = K.ca * as + K.cb * ps + K.cg * fs;
        op = K.ca * ap + K.cb * pv + K.cg * fp;
      } else {
        const double* sb = reinterpret_cast<const double*>(sl + SlotT::B);
        const double* sg = reinterpret_cast<const double*>(sl + SlotT::G);
        os = K.ca * as + K.cb * sm_half(sb, 0, lane) + K.cc * ps +
             K.cg * (K.cd * sm_half(sg, 0, lane) + K.ce * fs);
        op = K.ca * ap + K.cb * sm_half(sb, 1, lane) + K.cc * pv +
             K.cg * (K.cd * sm_half(sg, 1, lane) + K.ce * fp);
      }
    }
    if (active) {
      double* ob = reinterpret_cast<double*>(A.o + j * rs + chunk * kStateBlkDD) + h * 32 + lane;
      ob[0] = os.hi;
      ob[64] = op.hi;
      ob[128] = os.lo;
      ob[192] = op.lo;
      if (EPI == EPI_RK104_5) {
        double* fb = reinterpret_cast<double*>(A.f + j * rs + chunk * kStateBlkDD) + h * 32 + lane;
        fb[0] = fs.hi;
        fb[64] = fp.hi;
        fb[128] = fs.lo;
        fb[192] = fp.lo;
      }
      if (CHECK) bad |= !(fabs(os.hi) <= 1e30) || !(fabs(op.hi) <= 1e30);  // evolve.cpp:227-228
    }

    const int rn = j + 1 + R;
#pragma unroll
    for (int m = 0; m < SW - 1; ++m) wps[m] = wps[m + 1];
#pragma unroll
    for (int m = 0; m < PW - 1; ++m) wpi[m] = wpi[m + 1];
    if (rn >= n && A.phys_hi) {
      wps[SW - 1] = cubic_dd(wps[SW - 2], wps[SW - 3], wps[SW - 4], wps[SW - 5], K);
      wpi[PW - 1] = cubic_dd(wpi[PW - 2], wpi[PW - 3], wpi[PW - 4], wpi[PW - 5], K);
    } else {
      const double* sx = reinterpret_cast<const double*>(sl + SlotT::XN);
      wps[SW - 1] = sm_half(sx, 0, lane);
      wpi[PW - 1] = sm_half(sx, 1, lane);
    }
    __syncwarp();
    if (lane == 0 && j + S < je) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      issue(slot, j + S);
    }
    if (++slot == S) { slot = 0; parity ^= 1u; }
  }
  if (CHECK && __any_sync(kFull, bad) && lane == 0) {
    atomicExch(A.flag + 1, A.step >= 0 ? (unsigned long long)A.step : A.flag[2]);
    atomicOr(A.flag, 1ull);
  }
}

}  // namespace hwg
