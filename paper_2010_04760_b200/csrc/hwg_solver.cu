// Host runtime + C ABI of libhwgpu.so (include/hweno_gpu.h).
//
// The handle mirrors EvolutionRhs (proj/src/evolve.cpp:10-38) and the time
// loop advance_steps (evolve.cpp:237-265); the steppers' stage sequences are
// those of ssprk33_step / ssprk104_step (proj/include/hweno/timestep.hpp:54-109)
// with each stage one fused launch of hwg::stage_kernel (fp64 / mixed tiers)
// or hwg::stage_kernel_dd (double-double tiers).
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/hweno_gpu.h"
#include "hwg_launch.h"
#include <nvtx3/nvToolsExt.h>  // header-only NVTX v3: ranges for nsys / ncu --nvtx

using namespace hwg;

namespace {
thread_local std::string g_create_err;
}  // namespace
// hwg_last_error(NULL) of the handle-less entry points (hwg_coef.cu)
void hwg::set_global_error(const std::string& msg) { g_create_err = msg; }

namespace {
// NVTX range over a C-ABI entry point (no-op unless a profiler is attached)
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
};
}  // namespace

namespace {
// CUDA-graph cache entries per handle (least recently used goes first)
constexpr size_t kMaxGraphs = 8;
// fused halo push: minimum rows per rho range (max(IL, R, halo) over the schemes)
constexpr int kMinPeerRangeRows = 4;
// DD tiers: rows per rho range from which the mixed tier's inlined row loop
// is launched (hwg_stage_dd.cu, DDLauncher)
constexpr int kDDInlineRows = 400;

// Host double-double, an exact replica of the reference's DDReal operators
// (proj/include/hweno/precision.hpp:16-115).  Like the reference, the host
// side is compiled with -ffp-contract=off (build.py) so no multiply-add is
// fused; std::fma is explicit.
struct DD {
  double hi, lo;
};
inline double two_sum(double a, double b, double& e) {
  double s = a + b;
  double bb = s - a;
  e = (a - (s - bb)) + (b - bb);
  return s;
}
inline double quick_two_sum(double a, double b, double& e) {
  double s = a + b;
  e = b - (s - a);
  return s;
}
inline double two_prod(double a, double b, double& e) {
  double p = a * b;
  e = std::fma(a, b, -p);
  return p;
}
inline DD dd_add(DD a, DD b) {
  double s2, t2;
  double s1 = two_sum(a.hi, b.hi, s2);
  double t1 = two_sum(a.lo, b.lo, t2);
  s2 += t1;
  s1 = quick_two_sum(s1, s2, s2);
  s2 += t2;
  s1 = quick_two_sum(s1, s2, s2);
  return {s1, s2};
}
inline DD dd_addd(DD a, double b) {
  double s2;
  double s1 = two_sum(a.hi, b, s2);
  s2 += a.lo;
  s1 = quick_two_sum(s1, s2, s2);
  return {s1, s2};
}
inline DD dd_neg(DD a) { return {-a.hi, -a.lo}; }
inline DD dd_sub(DD a, DD b) { return dd_add(a, dd_neg(b)); }
inline DD dd_mul(DD a, DD b) {
  double p2;
  double p1 = two_prod(a.hi, b.hi, p2);
  p2 += a.hi * b.lo + a.lo * b.hi;
  p1 = quick_two_sum(p1, p2, p2);
  return {p1, p2};
}
inline DD dd_muld(DD a, double b) {
  double p2;
  double p1 = two_prod(a.hi, b, p2);
  p2 += a.lo * b;
  p1 = quick_two_sum(p1, p2, p2);
  return {p1, p2};
}
inline DD dd_div(DD a, DD b) {  // precision.hpp operator/
  double q1 = a.hi / b.hi;
  DD r = dd_sub(a, dd_muld(b, q1));
  double q2 = r.hi / b.hi;
  r = dd_sub(r, dd_muld(b, q2));
  double q3 = r.hi / b.hi;
  double s2;
  double s1 = quick_two_sum(q1, q2, s2);
  return dd_addd({s1, s2}, q3);
}
inline DD I(double v) { return {v, 0.0}; }
inline DD Q(double num, double den) { return dd_div(I(num), I(den)); }
inline dd to_dev(DD v) { return {v.hi, v.lo}; }
}  // namespace

struct hwg_solver {
  hwg_desc d{};
  bool ddm = false;          // double-double tier
  int n = 0, nt = 0, ntp = 0, phys_lo = 1, phys_hi = 1;
  int dev = 0;
  cudaStream_t stream = nullptr;
  cudaStream_t own = nullptr;
  int sblk = kStateBlk;      // double2 per (row, chunk) state block
  int cblk = kCoefBlk;       // double2 per (row, chunk) coefficient block
  double2* coef = nullptr;   // coefficient blocks
  DDConsts* kdev = nullptr;  // DD tiers: the reference's DD constants, device copy
  double* cot = nullptr;     // cot(theta) (fp64, or dd pairs), padded to nchunks*32
  double2* reg[5] = {};      // state registers, blocked layout incl. halo rows
  int nreg = 0;
  size_t rs = 0;             // double2 per state row (nchunks * sblk + pad)
  size_t crs = 0;            // double2 per coefficient row (nchunks * cblk + pad)
  size_t reg_elems = 0;      // double2 per register ((n + 2 kHalo) * rs)
  int cur = 0, scr1 = 1, scr2 = 2, scr3 = 3, scr4 = 4;
  unsigned long long* flag = nullptr;
  unsigned long long* hflag = nullptr;  // pinned
  int nchunks = 0, nranges = 0, blocks = 0, wpb = kWarpsPerBlock;
  double* stage_dev = nullptr;
  size_t stage_cap = 0;
  DD drho{0, 0}, dtheta{0, 0}, eps{0, 0}, sigma{0, 0};
  // CUDA graphs of one register-rotation period (2 steps), keyed by stepper,
  // dt and the rotation state at capture
  struct GraphEntry {
    int stepper;
    double dt_hi, dt_lo;
    int rot[5];
    cudaGraphExec_t exec;
  };
  std::vector<GraphEntry> graphs;
  bool use_graphs = true;
  bool use_pdl = true;       // programmatic dependent launch of the stage kernels
  bool abort_req = false;    // hwg_abort_advance called from the hook
  // observers
  int kobs = -1, j0 = -1, jobs = -1;
  double* obs_w = nullptr;   // 32 horizon weights + ntheta projection weights
  double* obs_dev = nullptr; // 14 outputs
  double* obs_host = nullptr;
  // fused halo push (hwg_set_peers)
  struct Peer {
    bool on = false;
    double2* reg[5] = {};
    unsigned long long* flag = nullptr;
    long long n = 0;
    std::vector<void*> opened;  // IPC mappings to close
  } plo, phi;
  long long peer_timeout_ns = 10000000000LL;
  std::string err;
};

#define CK(call)                                                               \
  do {                                                                         \
    cudaError_t e_ = (call);                                                   \
    if (e_ != cudaSuccess) {                                                   \
      s->err = std::string(#call) + ": " + cudaGetErrorString(e_);             \
      return HWG_ECUDA;                                                        \
    }                                                                          \
  } while (0)

// ----------------------------------------------------------------------------
// layout kernels
namespace hwg {

// host FieldLayout <-> device register (row 0 pointer), blocked; stride 2 =
// DD {hi, lo} pairs on the host.  dd: the register holds lo limbs at +64.
__global__ void relayout_kernel2(const double* __restrict__ src, double* __restrict__ dst,
                                 double2* reg, int n, int nt, size_t rs, int stride, int dir,
                                 int sblk) {
  __shared__ double tile[4][32][33];
  const int j0 = blockIdx.x * 32, k0 = blockIdx.y * 32;
  const int tx = threadIdx.x, ty = threadIdx.y;
  const size_t W = (size_t)n + 8, Hh = (size_t)nt + 4, P = W * Hh;
  const bool dd = sblk == kStateBlkDD;
  for (int limb = 0; limb < 2; ++limb) {
    if (limb == 1 && !dd && !(dir == 1 && stride == 2)) break;
    const int off = limb * 64;  // lo limbs at +64 in a DD block
    if (dir == 0) {
      for (int kk = ty; kk < 32; kk += 8) {
        const int k = k0 + kk, j = j0 + tx;
        if (k < nt && j < n)
          for (int c = 0; c < 4; ++c) {
            const size_t o = (c * P + (size_t)(k + 2) * W + (j + 4)) * stride;
            tile[c][kk][tx] = limb == 0 ? src[o] : (stride == 2 ? src[o + 1] : 0.0);
          }
      }
      __syncthreads();
      for (int jj = ty; jj < 32; jj += 8) {
        const int j = j0 + jj, k = k0 + tx;
        if (k < nt && j < n) {
          double2* b = reg + j * rs + (size_t)(k >> 5) * sblk + (k & 31) + off;
          b[0] = make_double2(tile[0][tx][jj], tile[1][tx][jj]);
          b[32] = make_double2(tile[2][tx][jj], tile[3][tx][jj]);
        }
      }
    } else {
      for (int jj = ty; jj < 32; jj += 8) {
        const int j = j0 + jj, k = k0 + tx;
        if (k < nt && j < n) {
          double2 u = make_double2(0.0, 0.0), v = u;
          if (limb == 0 || dd) {
            const double2* b = reg + j * rs + (size_t)(k >> 5) * sblk + (k & 31) + off;
            u = b[0];
            v = b[32];
          }
          tile[0][tx][jj] = u.x; tile[1][tx][jj] = u.y;
          tile[2][tx][jj] = v.x; tile[3][tx][jj] = v.y;
        }
      }
      __syncthreads();
      for (int kk = ty; kk < 32; kk += 8) {
        const int k = k0 + kk, j = j0 + tx;
        if (k < nt && j < n)
          for (int c = 0; c < 4; ++c)
            dst[(c * P + (size_t)(k + 2) * W + (j + 4)) * stride + limb] = tile[c][kk][tx];
      }
    }
    __syncthreads();
  }
}

// the reference's ghost rules (evolve.cpp:40-71) on an fp64 FieldLayout in
// device memory, same arithmetic as fill_host_ghosts (no contraction):
// blockIdx.y = 0: radial cubic continuation, one thread per (component, k);
// blockIdx.y = 1: theta parity images, one thread per (component, j)
__global__ void ghost_kernel(double* u, int n, int nt, int even) {
  const long long W = n + 8, P = W * (nt + 4);
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  auto at = [&](int c, int j, int k) -> double& { return u[c * P + (long long)(k + 2) * W + (j + 4)]; };
  auto cub = [](double a, double b, double c, double d) { return 4.0 * a - 6.0 * b + 4.0 * c - d; };
  if (blockIdx.y == 0) {
    if (i >= 4 * nt) return;
    const int c = i / nt, k = i % nt;
    for (int t = 1; t <= 4; ++t)
      at(c, -t, k) = cub(at(c, -t + 1, k), at(c, -t + 2, k), at(c, -t + 3, k), at(c, -t + 4, k));
    for (int t = 1; t <= 4; ++t)
      at(c, n - 1 + t, k) = cub(at(c, n - 2 + t, k), at(c, n - 3 + t, k), at(c, n - 4 + t, k),
                                at(c, n - 5 + t, k));
  } else {
    if (i >= 4 * n) return;
    const int c = i / n, j = i % n;
    for (int t = 0; t < 2; ++t) {
      const double north = at(c, j, t), south = at(c, j, nt - 1 - t);
      at(c, j, -1 - t) = even ? north : -north;
      at(c, j, nt + t) = even ? south : -south;
    }
  }
}

// coefficient plane q (index j + ld*k, rows row0..) -> blocked coefficient
// member, times `scale`; lo = 1 writes the DD low limbs (block offset kCoefBlk)
__global__ void coef_kernel(const double* __restrict__ src, int ld, int row0, double* coef,
                            int q, int n, int nt, int nchunks, int cblk, size_t crs, int lo,
                            double scale) {
  __shared__ double tile[32][33];
  const int j0 = blockIdx.x * 32, k0 = blockIdx.y * 32;
  const int tx = threadIdx.x, ty = threadIdx.y;
  for (int kk = ty; kk < 32; kk += 8) {
    const int k = k0 + kk, j = j0 + tx;
    if (k < nt && j < n) tile[kk][tx] = src[(size_t)(j + row0) + (size_t)ld * k];
  }
  __syncthreads();
  for (int jj = ty; jj < 32; jj += 8) {
    const int j = j0 + jj, k = k0 + tx;
    if (j < n && k < nchunks * 32) {
      const size_t blk = (size_t)j * crs + (size_t)(k >> 5) * cblk + (lo ? kCoefBlk : 0);
      size_t o;
      if (q < 8) o = (blk + (q / 2) * 32 + (k & 31)) * 2 + (q % 2);
      else o = (blk + kCoefAth) * 2 + (k & 31);
      coef[o] = (k < nt) ? tile[tx][jj] * scale : 0.0;
    }
  }
}

__global__ void observe_kernel2(const double2* reg, size_t rs, int sblk, int j0,
                                const double* hw, int kobs, int jobs, int jscri, const double* pw,
                                int nt, double* out) {
  auto psi = [&](int j, int k) { return reg[j * rs + (size_t)(k >> 5) * sblk + (k & 31)]; };
  const int lane = threadIdx.x;
  if (lane == 0) {
    // HorizonSampler::sample (diagnostics.cpp:145-160): sequential dot products
    for (int d = 0; d < 4; ++d) {
      double sr = 0.0, si = 0.0;
      if (j0 >= 0 && kobs >= 0)
        for (int i = 0; i < 5 + d; ++i) {
          const double2 v = psi(j0 + i, kobs);
          sr = sr + hw[d * 8 + i] * v.x;
          si = si + hw[d * 8 + i] * v.y;
        }
      out[2 * d] = sr;
      out[2 * d + 1] = si;
    }
    double2 o = (jobs >= 0 && kobs >= 0) ? psi(jobs, kobs) : make_double2(0, 0);
    out[8] = o.x; out[9] = o.y;
    double2 sc = (jscri >= 0 && kobs >= 0) ? psi(jscri, kobs) : make_double2(0, 0);
    out[10] = sc.x; out[11] = sc.y;
  }
  // multipole_project as a linear functional of the theta slice at jobs
  double pr = 0.0, pim = 0.0;
  if (jobs >= 0)
    for (int k = lane; k < nt; k += 32) {
      const double2 v = psi(jobs, k);
      pr = fma(pw[k], v.x, pr);
      pim = fma(pw[k], v.y, pim);
    }
  for (int o = 16; o > 0; o >>= 1) {
    pr += __shfl_xor_sync(kFull, pr, o);
    pim += __shfl_xor_sync(kFull, pim, o);
  }
  if (lane == 0) { out[12] = pr; out[13] = pim; }
}

}  // namespace hwg

// ----------------------------------------------------------------------------
namespace {

int mode_of(const hwg_solver* s) {
  if (s->d.scheme == HWG_FD6KO) return F64;  // no weights
  if (std::isinf(s->d.eps)) return LIN;
  const bool mixed = s->d.precision == HWG_MIXED || s->d.precision == HWG_DD_MIXED;
  return mixed ? MIXED : F64;
}

int launch(hwg_solver* s, const StageArgs& a, int epi, int blocks = 0) {
  launch_stage_fast(a, s->d.scheme, mode_of(s), epi, blocks > 0 ? blocks : s->blocks, s->wpb,
                    s->stream);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    s->err = std::string("stage launch: ") + cudaGetErrorString(e);
    return HWG_ECUDA;
  }
  return HWG_OK;
}

int launch(hwg_solver* s, const StageArgsDD& a, int epi) {
  launch_stage_dd(a, s->d.scheme, mode_of(s), epi, s->blocks, s->wpb, s->stream);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    s->err = std::string("stage launch: ") + cudaGetErrorString(e);
    return HWG_ECUDA;
  }
  return HWG_OK;
}

// row-0 pointer of state register r
double2* row0(const hwg_solver* s, int r) { return s->reg[r] + (size_t)kHalo * s->rs; }

// 1/(6 drho) (WENO5), 1/(2 drho) (WENO3), 1/(60 drho) (FD6): the factor of
// the radial differences, spatial.hpp:152, :178-182
double radial_scale(const hwg_solver* s) {
  const double dr = s->d.drho;
  if (s->d.scheme == HWG_WENO5) return 1.0 / (6.0 * dr);
  if (s->d.scheme == HWG_WENO3) return 1.0 / (2.0 * dr);
  return 1.0 / (60.0 * dr);
}
// 1/(12 dth^2): the second-derivative factor of the theta operator (spatial.hpp:212)
double theta_scale(const hwg_solver* s) {
  return 1.0 / (12.0 * s->d.dtheta * s->d.dtheta);
}

StageArgs base_args(const hwg_solver* s) {
  StageArgs a{};
  a.n = s->n; a.nt = s->nt; a.nchunks = s->nchunks;
  a.rs = (long long)s->rs; a.crs = (long long)s->crs;
  a.pdl = s->use_pdl ? 1 : 0;
  a.row_lo = 0;
  a.row_hi = s->n;
  a.defer = 0;
  a.phys_lo = s->phys_lo; a.phys_hi = s->phys_hi;
  a.nranges = s->nranges;
  a.negpar = s->d.parity < 0 ? 1 : 0;
  a.eps4 = 4.0 * s->d.eps;
  a.eps = s->d.eps;
  a.epsf = (float)s->d.eps;
  const double dr = s->d.drho;
  a.ko = s->d.sigma / (256.0 * dr);
  a.coef = s->coef;
  a.cot = s->cot;
  a.flag = s->flag;
  return a;
}

// the reference's per-call DD constants, evaluated once with its own DD ops
StageArgsDD base_args_dd(const hwg_solver* s) {
  StageArgsDD a{};
  a.n = s->n; a.nt = s->nt; a.nchunks = s->nchunks;
  a.phys_lo = s->phys_lo; a.phys_hi = s->phys_hi;
  a.nranges = s->nranges;
  a.negpar = s->d.parity < 0 ? 1 : 0;
  a.eps_hi = s->eps.hi;  // demote(spec_.eps), evolve.cpp:79-80
  // long rho ranges: the mixed tier's row-loop interfaces inlined (+5 % at
  // 885 rows per range; -2..-9 % at 14-55 rows, profiles/r02_dd_ab2.txt)
  a.inl = s->n >= kDDInlineRows * s->nranges ? 1 : 0;
  if (const char* e = std::getenv("HWG_DD_INL")) a.inl = std::atoi(e);
  a.cot = reinterpret_cast<const dd*>(s->cot);
  a.coef = s->coef;
  a.flag = s->flag;
  a.kdev = s->kdev;
  DDConsts& K = a.k;
  K.c1312 = to_dev(Q(13, 12));
  K.quarter = to_dev(Q(1, 4));
  K.d0 = to_dev(Q(1, 10)); K.d1 = to_dev(Q(6, 10)); K.d2 = to_dev(Q(3, 10));
  K.one = to_dev(I(1));
  K.sixth = to_dev(Q(1, 6));
  K.third = to_dev(Q(1, 3)); K.twothird = to_dev(Q(2, 3));
  K.half = to_dev(Q(1, 2));
  K.inv_drho = to_dev(dd_div(I(1), s->drho));                                  // spatial.hpp:143
  K.inv1 = to_dev(dd_div(I(1), dd_mul(I(12), s->dtheta)));                     // :211
  K.inv2 = to_dev(dd_div(I(1), dd_mul(dd_mul(I(12), s->dtheta), s->dtheta)));  // :212
  K.eps = to_dev(s->eps);
  K.sigma = to_dev(s->sigma);
  K.h60 = to_dev(dd_mul(I(60), s->drho));
  K.h256 = to_dev(dd_mul(I(256), s->drho));
  const double ints[16] = {4, 6, 9, 45, 8, 28, 56, 70, 16, 30, 12, 2, 3, 5, 7, 11};
  dd* iv[16] = {&K.c4, &K.c6, &K.c9, &K.c45, &K.c8, &K.c28, &K.c56, &K.c70,
                &K.c16, &K.c30, &K.c12, &K.c2, &K.c3, &K.c5, &K.c7, &K.c11};
  for (int i = 0; i < 16; ++i) *iv[i] = to_dev(I(ints[i]));
  const bool full = s->d.precision == HWG_DD_FULL;
  // eps = inf weights in the weight scalar TW (spatial.hpp:33-38, 100-103)
  K.lw5[0] = full ? to_dev(Q(1, 10)) : to_dev(I(1.0 / 10.0));
  K.lw5[1] = full ? to_dev(Q(6, 10)) : to_dev(I(6.0 / 10.0));
  K.lw5[2] = full ? to_dev(Q(3, 10)) : to_dev(I(3.0 / 10.0));
  K.lw3[0] = full ? to_dev(Q(1, 3)) : to_dev(I(1.0 / 3.0));
  K.lw3[1] = full ? to_dev(Q(2, 3)) : to_dev(I(2.0 / 3.0));
  return a;
}

int ensure_regs(hwg_solver* s, int need) {
  while (s->nreg < need) {
    double2* p = nullptr;
    CK(cudaMalloc(&p, s->reg_elems * sizeof(double2)));
    CK(cudaMemsetAsync(p, 0, s->reg_elems * sizeof(double2), s->stream));
    s->reg[s->nreg++] = p;
  }
  return HWG_OK;
}

// stage-input register for (stepper, stage) given the current rotation
int stage_input_reg(const hwg_solver* s, int stepper, int stage) {
  if (stepper == HWG_SSPRK33) {
    const int in[3] = {s->cur, s->scr1, s->scr2};
    return in[stage];
  }
  // rk104: U=cur, P=scr1, Q=scr2, S4=scr3, F4=scr4
  const int P = s->scr1, Qr = s->scr2, S4 = s->scr3;
  const int in[10] = {s->cur, P, Qr, P, S4, P, Qr, P, Qr, P};
  return in[stage];
}

// Stage plan shared by both tiers: registers and RK constants
// (timestep.hpp:61-70 for ssprk33, :84-108 for ssprk104 with u^(4) kept in
// its own register instead of a copy).  Constants in DD (the fp64 tier uses .hi).
struct Plan {
  int x, out, ua = -1, ub = -1, ug = -1, f = -1, epi;
  DD ca{0, 0}, cb{0, 0}, cc{0, 0}, cg{0, 0}, cd{0, 0}, ce{0, 0};
  int rot = 0;  // 1: swap cur<->scr1 after, 2: swap cur<->scr2 after
};

Plan make_plan(const hwg_solver* s, int stepper, int stage, DD dt) {
  Plan p{};
  if (stepper == HWG_SSPRK33) {
    if (stage == 0) {
      p.x = s->cur; p.out = s->scr1; p.cg = dt; p.epi = EPI_AXPY;
    } else if (stage == 1) {
      p.x = s->scr1; p.out = s->scr2; p.ua = s->cur; p.epi = EPI_RK3;
      p.ca = Q(3, 4); p.cb = Q(1, 4); p.cg = dt;
    } else {
      p.x = s->scr2; p.out = s->scr1; p.ua = s->cur; p.epi = EPI_RK3C;
      p.ca = Q(1, 3); p.cb = Q(2, 3); p.cg = dt; p.rot = 1;
    }
    return p;
  }
  const int U = s->cur, P = s->scr1, Qr = s->scr2, S4 = s->scr3, F4 = s->scr4;
  const int ins[10] = {U, P, Qr, P, S4, P, Qr, P, Qr, P};
  const int outs[10] = {P, Qr, P, S4, P, Qr, P, Qr, P, Qr};
  p.x = ins[stage];
  p.out = outs[stage];
  if (stage == 4) {
    p.ua = U; p.f = F4; p.epi = EPI_RK104_5;
    p.ca = Q(3, 5); p.cb = Q(2, 5); p.cg = dd_div(dt, I(15));
  } else if (stage == 9) {
    p.ua = U; p.ub = S4; p.ug = F4; p.epi = EPI_RK104_10;
    p.ca = Q(1, 25); p.cb = Q(9, 25); p.cc = Q(3, 5);
    p.cg = dt; p.cd = Q(3, 50); p.ce = Q(1, 10); p.rot = 2;
  } else {
    p.epi = EPI_AXPY; p.cg = dd_div(dt, I(6));
  }
  return p;
}

// rows a neighbour reads across the slab edge (slabs.py HALO_ROWS)
int halo_rows(int scheme) { return scheme == HWG_WENO5 ? 3 : scheme == HWG_WENO3 ? 2 : 4; }

// step >= 0: the kernel records step + 1 on blow-up; step < 0: counter mode
// (flag[2] is bumped by stage 0 and recorded by the scan) for graph replay
// One stage, or one part of it: rows [row_lo, row_hi) (fast tiers; the
// double-double tiers always run whole stages).  `first`: the part that
// bumps the device step counter; `last`: the part that publishes the blow-up
// bit and rotates the registers.
int do_stage_part(hwg_solver* s, int stepper, int stage, double dt_hi, double dt_lo,
                  long long step, int row_lo, int row_hi, bool first, bool last);

int do_stage(hwg_solver* s, int stepper, int stage, double dt_hi, double dt_lo, long long step) {
  return do_stage_part(s, stepper, stage, dt_hi, dt_lo, step, 0, s->n, true, true);
}

// kernel arguments of one fast-tier stage (or one part of it: rows
// [row_lo, row_hi)); *blocks_out: the launch's grid (0 = the handle's)
StageArgs fast_stage_args(const hwg_solver* s, const Plan& p, int stage, long long step,
                        int row_lo, int row_hi, bool first, bool last, int* blocks_out) {
  const long long rec = step >= 0 ? step + 1 : -1;
  const int bump = (step < 0 && stage == 0 && first) ? 1 : 0;
  auto r0 = [&](int r) -> double2* { return r >= 0 ? row0(s, r) : nullptr; };
  StageArgs a = base_args(s);
  a.step = rec;
  a.bump = bump;
  a.x = r0(p.x); a.o = r0(p.out); a.ua = r0(p.ua); a.ub = r0(p.ub); a.ug = r0(p.ug);
  a.f = r0(p.f);
  a.ca = p.ca.hi; a.cb = p.cb.hi; a.cc = p.cc.hi; a.cg = p.cg.hi; a.cd = p.cd.hi; a.ce = p.ce.hi;
  const bool check = p.epi == EPI_RK3C || p.epi == EPI_RK104_10;
  if (s->plo.on || s->phi.on) {
    PeerArgs& x = a.px;
    x.h = halo_rows(s->d.scheme);
    x.wait = s->flag + 6;
    x.epoch = s->flag + 5;
    x.timeout_ns = s->peer_timeout_ns;
    if (s->plo.on) {
      x.on_lo = 1;
      x.o_lo = s->plo.reg[p.out] + (size_t)(kHalo + s->plo.n) * s->rs;
      x.sig_lo = s->plo.flag + 7;
    }
    if (s->phi.on) {
      x.on_hi = 1;
      x.o_hi = s->phi.reg[p.out] + (size_t)(kHalo - x.h) * s->rs;
      x.sig_hi = s->phi.flag + 6;
    }
  }
  int blocks = 0;
  if (s->plo.on || s->phi.on) {
    // fused halo push: only the first and last range wait for the
    // neighbours' rows and only they push, so every range must span at
    // least max(IL, R, h) = 4 rows — then no other range's window reaches
    // a halo row and ranges 0 / last own the pushed output rows
    a.nranges = std::min(s->nranges, std::max(1, s->n / kMinPeerRangeRows));
    blocks = (int)(((long long)a.nranges * s->nchunks + s->wpb - 1) / s->wpb);
  }
  if (row_lo != 0 || row_hi != s->n) {  // a part: ranges in proportion to its rows
    a.row_lo = row_lo;
    a.row_hi = row_hi;
    const int span = row_hi - row_lo;
    a.nranges = (int)std::max<long long>(
        1, std::min<long long>((long long)s->nranges * span / s->n, span / 2));
    blocks = (int)(((long long)a.nranges * s->nchunks + s->wpb - 1) / s->wpb);
  }
  if (last && (check || s->plo.on || s->phi.on)) a.tick = s->flag + 4;
  if (!last && check) a.defer = 1;
  *blocks_out = blocks;
  return a;
}

int do_stage_part(hwg_solver* s, int stepper, int stage, double dt_hi, double dt_lo,
                  long long step, int row_lo, int row_hi, bool first, bool last) {
  const Plan p = make_plan(s, stepper, stage, DD{dt_hi, dt_lo});
  const long long rec = step >= 0 ? step + 1 : -1;
  const int bump = (step < 0 && stage == 0 && first) ? 1 : 0;
  int rc;
  auto r0 = [&](int r) -> double2* { return r >= 0 ? row0(s, r) : nullptr; };
  if (s->ddm) {
    StageArgsDD a = base_args_dd(s);
    a.step = rec;
    a.bump = bump;
    a.x = r0(p.x); a.o = r0(p.out); a.ua = r0(p.ua); a.ub = r0(p.ub); a.ug = r0(p.ug);
    a.f = r0(p.f);
    a.k.ca = to_dev(p.ca); a.k.cb = to_dev(p.cb); a.k.cc = to_dev(p.cc);
    a.k.cg = to_dev(p.cg); a.k.cd = to_dev(p.cd); a.k.ce = to_dev(p.ce);
    rc = launch(s, a, p.epi);
  } else {
    int blocks = 0;
    const StageArgs a = fast_stage_args(s, p, stage, step, row_lo, row_hi, first, last, &blocks);
    rc = launch(s, a, p.epi, blocks);
  }
  // the host's register rotation follows the device only for launched stages
  if (rc == HWG_OK && last && p.rot == 1) std::swap(s->cur, s->scr1);
  if (rc == HWG_OK && last && p.rot == 2) std::swap(s->cur, s->scr2);
  return rc;
}

int ensure_staging(hwg_solver* s, size_t cnt) {
  if (s->stage_cap < cnt) {
    if (s->stage_dev) cudaFree(s->stage_dev);
    s->stage_dev = nullptr;
    s->stage_cap = 0;
    CK(cudaMalloc(&s->stage_dev, cnt * sizeof(double)));
    s->stage_cap = cnt;
  }
  return HWG_OK;
}

int upload_layout(hwg_solver* s, const double* host, int stride, int reg) {
  const size_t cnt = (size_t)4 * (s->n + 8) * (s->nt + 4) * stride;
  int rc = ensure_staging(s, cnt);
  if (rc) return rc;
  CK(cudaMemcpyAsync(s->stage_dev, host, cnt * sizeof(double), cudaMemcpyHostToDevice, s->stream));
  dim3 grid((s->n + 31) / 32, (s->nt + 31) / 32), blk(32, 8);
  relayout_kernel2<<<grid, blk, 0, s->stream>>>(s->stage_dev, nullptr, row0(s, reg), s->n, s->nt,
                                                 s->rs, stride, 0, s->sblk);
  CK(cudaGetLastError());
  return HWG_OK;
}

// the reference's ghost rules (evolve.cpp:40-71) on a host FieldLayout, in
// fp64 or (stride 2) in double-double with the reference's DD operators
void fill_host_ghosts(const hwg_solver* s, double* u, int stride, bool dd_arith) {
  const int n = s->n, nt = s->nt;
  const long long W = n + 8, P = W * (nt + 4);
  auto idx = [&](int c, int j, int k) { return (c * P + (long long)(k + 2) * W + (j + 4)) * stride; };
  auto get = [&](int c, int j, int k) -> DD {
    const long long o = idx(c, j, k);
    return {u[o], stride == 2 ? u[o + 1] : 0.0};
  };
  auto put = [&](int c, int j, int k, DD v) {
    const long long o = idx(c, j, k);
    u[o] = v.hi;
    if (stride == 2) u[o + 1] = v.lo;
  };
  auto cub = [&](DD a, DD b, DD c, DD d) -> DD {
    if (dd_arith)  // WorkReal(4) * p - WorkReal(6) * q + WorkReal(4) * r - t
      return dd_sub(dd_add(dd_sub(dd_mul(I(4), a), dd_mul(I(6), b)), dd_mul(I(4), c)), d);
    return I(4.0 * a.hi - 6.0 * b.hi + 4.0 * c.hi - d.hi);
  };
  for (int k = 0; k < nt; ++k)
    for (int c = 0; c < 4; ++c) {
      for (int t = 1; t <= 4; ++t)
        put(c, -t, k, cub(get(c, -t + 1, k), get(c, -t + 2, k), get(c, -t + 3, k), get(c, -t + 4, k)));
      for (int t = 1; t <= 4; ++t)
        put(c, n - 1 + t, k,
            cub(get(c, n - 2 + t, k), get(c, n - 3 + t, k), get(c, n - 4 + t, k), get(c, n - 5 + t, k)));
    }
  const bool even = s->d.parity > 0;
  for (int j = 0; j < n; ++j)
    for (int c = 0; c < 4; ++c)
      for (int t = 0; t < 2; ++t) {
        const DD north = get(c, j, t), south = get(c, j, nt - 1 - t);
        put(c, j, -1 - t, even ? north : dd_neg(north));
        put(c, j, nt + t, even ? south : dd_neg(south));
      }
}

// interior of register reg -> host FieldLayout (+ the reference's ghost rules)
int download_layout(hwg_solver* s, double* host, int stride, int reg, bool ghosts) {
  const size_t cnt = (size_t)4 * (s->n + 8) * (s->nt + 4) * stride;
  int rc = ensure_staging(s, cnt);
  if (rc) return rc;
  CK(cudaMemsetAsync(s->stage_dev, 0, cnt * sizeof(double), s->stream));
  dim3 grid((s->n + 31) / 32, (s->nt + 31) / 32), blk(32, 8);
  relayout_kernel2<<<grid, blk, 0, s->stream>>>(nullptr, s->stage_dev, row0(s, reg), s->n, s->nt,
                                                 s->rs, stride, 1, s->sblk);
  CK(cudaGetLastError());
  const bool dev_ghosts = ghosts && stride == 1;  // fp64 FieldLayout: ghosts on the device
  if (dev_ghosts) {
    const int m = 4 * std::max(s->n, s->nt);
    ghost_kernel<<<dim3((m + 255) / 256, 2), 256, 0, s->stream>>>(s->stage_dev, s->n, s->nt,
                                                                   s->d.parity > 0);
    CK(cudaGetLastError());
  }
  CK(cudaMemcpyAsync(host, s->stage_dev, cnt * sizeof(double), cudaMemcpyDeviceToHost, s->stream));
  CK(cudaStreamSynchronize(s->stream));
  if (ghosts && !dev_ghosts) fill_host_ghosts(s, host, stride, s->ddm && stride == 2);
  return HWG_OK;
}

int rhs_impl(hwg_solver* s, double* u, double* du, int stride) {
  int rc = upload_layout(s, u, stride, s->scr1);
  if (rc) return rc;
  if (s->ddm) {
    StageArgsDD a = base_args_dd(s);
    a.flag = nullptr;  // the RHS never freezes
    a.x = row0(s, s->scr1);
    a.o = row0(s, s->scr2);
    rc = launch(s, a, EPI_RHS);
  } else {
    StageArgs a = base_args(s);
    a.flag = nullptr;
    a.x = row0(s, s->scr1);
    a.o = row0(s, s->scr2);
    rc = launch(s, a, EPI_RHS);
  }
  if (rc) return rc;
  // du interior only; its ghosts stay as the caller gave them
  const int n = s->n, nt = s->nt;
  const size_t cnt = (size_t)4 * (n + 8) * (nt + 4) * stride;
  std::vector<double> tmp(cnt);
  rc = download_layout(s, tmp.data(), stride, s->scr2, false);
  if (rc) return rc;
  const long long W = n + 8, P = W * (nt + 4);
  for (int c = 0; c < 4; ++c)
    for (int k = 0; k < nt; ++k) {
      const size_t o = (c * P + (long long)(k + 2) * W + 4) * stride;
      std::memcpy(du + o, tmp.data() + o, sizeof(double) * n * stride);
    }
  fill_host_ghosts(s, u, stride, s->ddm && stride == 2);
  return HWG_OK;
}

DD tau_of(long long step, double dt_hi, double dt_lo) {  // WorkReal(double(s)) * dt
  return dd_mul(I((double)step), {dt_hi, dt_lo});
}

__global__ void set_counter_kernel(unsigned long long* ctr, long long v) { *ctr = (unsigned long long)v; }

bool graphs_ok(const hwg_solver* s) {
  if (!s->use_graphs || s->stream == nullptr || s->stream == cudaStreamLegacy ||
      s->stream == cudaStreamPerThread)
    return false;
  return true;
}

// nsteps whole steps from step_begin.  With graphs: the step counter is set
// once, then each pair of steps (one rotation period) replays a cached graph.
int launch_steps_impl(hwg_solver* s, int stepper, double dt_hi, double dt_lo, long long s0,
                      long long nsteps) {
  const int ns = stepper == HWG_SSPRK33 ? 3 : 10;
  if (stepper == HWG_SSPRK104) {
    int rc = ensure_regs(s, 5);
    if (rc) return rc;
  }
  // one whole step: ns stage launches (a single cooperative launch of all
  // three RK3 stages with neighbour dataflow was measured slower)
  auto one_step = [&](long long step) -> int {
    for (int st = 0; st < ns; ++st) {
      const int rc = do_stage(s, stepper, st, dt_hi, dt_lo, step);
      if (rc) return rc;
    }
    return HWG_OK;
  };
  if (!graphs_ok(s) || nsteps < 2) {
    for (long long q = 0; q < nsteps; ++q) {
      const int rc = one_step(s0 + q);
      if (rc) return rc;
    }
    return HWG_OK;
  }
  set_counter_kernel<<<1, 1, 0, s->stream>>>(s->flag + 2, s0);
  CK(cudaGetLastError());
  long long q = 0;
  for (; q + 2 <= nsteps; q += 2) {
    const int rot[5] = {s->cur, s->scr1, s->scr2, s->scr3, s->scr4};
    cudaGraphExec_t exec = nullptr;
    auto exec_it = s->graphs.end();
    for (auto it = s->graphs.begin(); it != s->graphs.end(); ++it)
      if (it->stepper == stepper && it->dt_hi == dt_hi && it->dt_lo == dt_lo &&
          std::equal(rot, rot + 5, it->rot)) {
        exec = it->exec;
        exec_it = it;
        break;
      }
    if (!exec) {
      cudaGraph_t g = nullptr;
      CK(cudaStreamBeginCapture(s->stream, cudaStreamCaptureModeThreadLocal));
      int rc = HWG_OK;
      for (int k = 0; k < 2 && rc == HWG_OK; ++k) rc = one_step(-1);
      cudaError_t ce = cudaStreamEndCapture(s->stream, &g);
      if (rc != HWG_OK || ce != cudaSuccess) {
        // nothing of the capture ran: drop it and undo its host bookkeeping
        if (g) cudaGraphDestroy(g);
        s->cur = rot[0]; s->scr1 = rot[1]; s->scr2 = rot[2]; s->scr3 = rot[3]; s->scr4 = rot[4];
        if (rc != HWG_OK) return rc;
        s->err = std::string("graph capture: ") + cudaGetErrorString(ce);
        return HWG_ECUDA;
      }
      cudaError_t ie = cudaGraphInstantiate(&exec, g, 0);
      cudaGraphDestroy(g);
      if (ie != cudaSuccess) {
        s->cur = rot[0]; s->scr1 = rot[1]; s->scr2 = rot[2]; s->scr3 = rot[3]; s->scr4 = rot[4];
        s->err = std::string("graph instantiate: ") + cudaGetErrorString(ie);
        return HWG_ECUDA;
      }
      // the capture ran do_stage's host bookkeeping for 2 steps: the
      // rotation is back where it started, as after a replay.  The cache is
      // keyed by dt: an adaptive-dt caller would grow it without bound, so
      // the least recently used entry goes once kMaxGraphs are held.
      if (s->graphs.size() >= kMaxGraphs) {
        cudaGraphExecDestroy(s->graphs.front().exec);
        s->graphs.erase(s->graphs.begin());
      }
      hwg_solver::GraphEntry e{stepper, dt_hi, dt_lo, {rot[0], rot[1], rot[2], rot[3], rot[4]}, exec};
      s->graphs.push_back(e);
    } else if (exec_it + 1 != s->graphs.end()) {
      // most recently used at the back
      hwg_solver::GraphEntry e = *exec_it;
      s->graphs.erase(exec_it);
      s->graphs.push_back(e);
    }
    CK(cudaGraphLaunch(exec, s->stream));
  }
  for (; q < nsteps; ++q) {
    const int rc = one_step(-1);
    if (rc) return rc;
  }
  return HWG_OK;
}

int create_impl(const hwg_desc* d, const double* coef, const double* coef_lo, const double* cotth,
                const double* cot_lo, bool ddm, hwg_solver** out) {
  *out = nullptr;
  if (!d || !coef || !cotth) {
    g_create_err = "hwg_create: null argument";
    return HWG_EINVAL;
  }
  // EvolutionRhs ctor: grid below stencil support (evolve.cpp:16-17)
  const int nglob = d->nrho_global > 0 ? d->nrho_global : d->nrho;
  if (nglob < 9 || d->ntheta < 2 || d->nrho < 8) {
    g_create_err = "EvolutionRhs: grid below stencil support";
    return HWG_EINVAL;
  }
  const bool prec_ok = ddm ? (d->precision == HWG_DD_FULL || d->precision == HWG_DD_MIXED)
                           : (d->precision == HWG_F64 || d->precision == HWG_MIXED);
  if (d->scheme < 0 || d->scheme > 2 || !prec_ok || !(d->drho > 0.0) || !(d->dtheta > 0.0)) {
    g_create_err = "hwg_create: invalid scheme/precision/spacing";
    return HWG_EINVAL;
  }
  const int ld = d->coef_ld > 0 ? d->coef_ld : nglob;
  const int row0_ = d->coef_row0 >= 0 ? d->coef_row0 : d->rho_offset;
  // lam sign structure (evolve.cpp:19-30): lam < 0 on [0, split), >= 0 after
  const double* lam = coef + (size_t)ld * d->ntheta;
  for (int k = 0; k < d->ntheta; ++k) {
    int j = 0;
    while (j < d->nrho && lam[(size_t)(row0_ + j) + (size_t)ld * k] < 0.0) ++j;
    for (; j < d->nrho; ++j)
      if (lam[(size_t)(row0_ + j) + (size_t)ld * k] < 0.0) {
        g_create_err = "EvolutionRhs: lam changes sign more than once along a row";
        return HWG_ERUNTIME;
      }
  }
  auto* s = new hwg_solver();
  s->d = *d;
  s->ddm = ddm;
  s->d.nrho_global = nglob;
  s->n = d->nrho;
  s->nt = d->ntheta;
  s->ntp = (d->ntheta + 31) / 32 * 32;
  s->nchunks = s->ntp / 32;
  s->sblk = ddm ? kStateBlkDD : kStateBlk;
  s->cblk = ddm ? kCoefBlkDD : kCoefBlk;
  // row pitches: the fast tiers may pad rows (HWG_STATE_PAD / HWG_COEF_PAD,
  // in double2) to spread concurrent row accesses over the HBM channels
  {
    size_t sp = 0, cp = 0;
    if (!ddm) {
      if (const char* e = std::getenv("HWG_STATE_PAD")) sp = (size_t)std::max(0, std::atoi(e));
      if (const char* e = std::getenv("HWG_COEF_PAD")) cp = (size_t)std::max(0, std::atoi(e));
    }
    s->rs = (size_t)s->nchunks * s->sblk + sp;
    s->crs = (size_t)s->nchunks * s->cblk + cp;
  }
  s->phys_lo = d->rho_offset == 0;
  s->phys_hi = d->rho_offset + d->nrho == nglob;
  s->dev = d->device;
  s->reg_elems = (size_t)(s->n + 2 * kHalo) * s->rs;
  s->drho = {d->drho, ddm ? d->drho_lo : 0.0};
  s->dtheta = {d->dtheta, ddm ? d->dtheta_lo : 0.0};
  s->eps = {d->eps, ddm ? d->eps_lo : 0.0};
  s->sigma = {d->sigma, ddm ? d->sigma_lo : 0.0};
  if (const char* e = std::getenv("HWG_NO_GRAPH")) s->use_graphs = e[0] == '0';
  if (const char* e = std::getenv("HWG_NO_PDL")) s->use_pdl = e[0] == '0';
  auto fail = [&](int rc) {
    g_create_err = s->err;
    hwg_destroy(s);
    return rc;
  };
  if (cudaSetDevice(s->dev) != cudaSuccess) {
    s->err = "cudaSetDevice failed (no GPU?)";
    return fail(HWG_ECUDA);
  }
#undef CK
#define CK(call)                                                               \
  do {                                                                         \
    cudaError_t e_ = (call);                                                   \
    if (e_ != cudaSuccess) {                                                   \
      s->err = std::string(#call) + ": " + cudaGetErrorString(e_);             \
      return fail(HWG_ECUDA);                                                  \
    }                                                                          \
  } while (0)
  CK(cudaStreamCreateWithFlags(&s->own, cudaStreamNonBlocking));
  s->stream = s->own;
  const size_t CB = (size_t)s->n * s->crs;
  CK(cudaMalloc(&s->coef, CB * sizeof(double2)));
  CK(cudaMemsetAsync(s->coef, 0, CB * sizeof(double2), s->stream));
  CK(cudaMalloc(&s->cot, 2 * s->ntp * sizeof(double)));
  // [0] blown (bit 1: peer timeout) [1] blowup step [2] step counter [3] pending
  // blow-up [4] launch ticket [5] peer epoch [6] / [7] arrivals from lower / upper
  // [0] blown [1] blow-up step [2] step counter [3] pending [4] ticket [5] peer
  // epoch [6,7] peer arrivals from lower / upper [8] peer waits that spun
  CK(cudaMalloc(&s->flag, 16 * sizeof(unsigned long long)));
  CK(cudaMemsetAsync(s->flag, 0, 16 * sizeof(unsigned long long), s->stream));
  CK(cudaMallocHost(&s->hflag, 2 * sizeof(unsigned long long)));
  CK(cudaMallocHost(&s->obs_host, 16 * sizeof(double)));
  CK(cudaMalloc(&s->obs_dev, 16 * sizeof(double)));
  CK(cudaMalloc(&s->obs_w, (32 + s->ntp) * sizeof(double)));
  CK(cudaMemsetAsync(s->obs_w, 0, (32 + s->ntp) * sizeof(double), s->stream));
  // coefficients: upload each reference plane (rows of this handle) and
  // transpose on the device into the blocked layout
  {
    double* tmp = nullptr;
    const size_t plane_src = (size_t)ld * s->nt;
    CK(cudaMalloc(&tmp, plane_src * sizeof(double)));
    dim3 grid((s->n + 31) / 32, s->nchunks), blk(32, 8);
    for (int limb = 0; limb < (ddm ? 2 : 1); ++limb) {
      const double* src = limb ? coef_lo : coef;
      for (int q = 0; q < 9; ++q) {
        if (src) {
          CK(cudaMemcpyAsync(tmp, src + q * plane_src, plane_src * sizeof(double),
                             cudaMemcpyHostToDevice, s->stream));
        } else {
          CK(cudaMemsetAsync(tmp, 0, plane_src * sizeof(double), s->stream));
        }
        // fast tiers: the radial derivative scale is folded into the planes
        // that multiply radial derivatives (b, lam, w) and the theta scale
        // 1/(12 dth^2) into ath (stage_body); the DD tiers keep the planes
        const double sc = ddm ? 1.0 : (q < 4 ? radial_scale(s) : q == 8 ? theta_scale(s) : 1.0);
        coef_kernel<<<grid, blk, 0, s->stream>>>(tmp, ld, row0_, reinterpret_cast<double*>(s->coef),
                                                  q, s->n, s->nt, s->nchunks, s->cblk, s->crs, limb,
                                                  sc);
        CK(cudaGetLastError());
      }
    }
    CK(cudaStreamSynchronize(s->stream));
    cudaFree(tmp);
    std::vector<double> c(2 * s->ntp, 0.0);
    for (int k = 0; k < s->nt; ++k) {
      if (ddm) {
        c[2 * k] = cotth[k];
        c[2 * k + 1] = cot_lo ? cot_lo[k] : 0.0;
      } else {
        c[k] = cotth[k] * s->d.dtheta;  // cot * (1/(12 dth)) / (1/(12 dth^2))
      }
    }
    CK(cudaMemcpy(s->cot, c.data(), 2 * s->ntp * sizeof(double), cudaMemcpyHostToDevice));
  }
  {
    int rc = ensure_regs(s, 3);
    if (rc) return fail(rc);
  }
  if (ddm) {
    CK(cudaMalloc(&s->kdev, sizeof(DDConsts)));
    const DDConsts k = base_args_dd(s).k;
    CK(cudaMemcpy(s->kdev, &k, sizeof(DDConsts), cudaMemcpyHostToDevice));
  }
  // launch geometry: one wave of warps, rho ranges balanced per theta chunk
  {
    int nsm = 148, occ = 1;
    CK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, s->dev));
    CK(ddm ? occupancy_dd(&occ) : occupancy_fast(&occ, mode_of(s)));
    // work units: one warp per (theta chunk, rho range)
    const int upb = kWarpsPerBlock;
    const long long target = (long long)nsm * std::max(occ, 1) * upb;
    const int wpc = ddm ? dd_warps_per_chunk() : 1;  // warps per theta chunk
    long long nr = std::max<long long>(1, target / ((long long)s->nchunks * wpc));
    // rows per range: as few as 2 on tiny grids to fill the wave (the window
    // warm-up costs ~2 rows of work, so larger grids keep longer ranges)
    // (the double-double kernel's window set-up assumes ranges of >= 4 rows)
    int minrows = ddm ? 4 : 2;
    if (const char* e = std::getenv("HWG_MIN_ROWS")) minrows = std::max(minrows, std::atoi(e));
    nr = std::min<long long>(nr, std::max(1, s->n / minrows));
    s->nranges = (int)nr;
    // small grids: fewer warps per block so the warps spread over all SMs
    const long long units = nr * s->nchunks * wpc;
    s->wpb = upb;  // warps per block
    while (s->wpb > 1 && units / s->wpb < nsm) s->wpb /= 2;
    s->blocks = (int)((units + s->wpb - 1) / s->wpb);
  }

  CK(cudaStreamSynchronize(s->stream));
#undef CK
#define CK(call)                                                               \
  do {                                                                         \
    cudaError_t e_ = (call);                                                   \
    if (e_ != cudaSuccess) {                                                   \
      s->err = std::string(#call) + ": " + cudaGetErrorString(e_);             \
      return HWG_ECUDA;                                                        \
    }                                                                          \
  } while (0)
  *out = s;
  return HWG_OK;
}

}  // namespace

// ----------------------------------------------------------------------------
// No C++ exception crosses the C ABI: every entry point runs under
// guarded(), which maps std::bad_alloc / std::exception to HWG_ERUNTIME
// with the message in hwg_last_error (int status returns).
template <class S>
void set_err(S* s, const char* msg) noexcept {
  try {
    if (s) const_cast<hwg_solver*>(s)->err = msg;
    else g_create_err = msg;
  } catch (...) {
  }
}
template <class S, class F>
int guarded(S* s, F&& f) noexcept {
  try {
    return f();
  } catch (const std::bad_alloc&) {
    set_err(s, "out of host memory");
  } catch (const std::exception& e) {
    set_err(s, e.what());
  } catch (...) {
    set_err(s, "unknown C++ exception");
  }
  return HWG_ERUNTIME;
}

extern "C" {

const char* hwg_last_error(const hwg_solver* s) {
  return s ? s->err.c_str() : g_create_err.c_str();
}

int hwg_create(const hwg_desc* d, const double* coef, const double* cotth, hwg_solver** out) {
  return guarded(static_cast<hwg_solver*>(nullptr), [&]() -> int {
    NvtxRange nvtx_("hwg_create");
    return create_impl(d, coef, nullptr, cotth, nullptr, false, out);
  });
}

int hwg_create_dd(const hwg_desc* d, const double* coef_hi, const double* coef_lo,
                  const double* cot_hi, const double* cot_lo, hwg_solver** out) {
  return guarded(static_cast<hwg_solver*>(nullptr), [&]() -> int {
    NvtxRange nvtx_("hwg_create_dd");
    return create_impl(d, coef_hi, coef_lo, cot_hi, cot_lo, true, out);
  });
}

void hwg_destroy(hwg_solver* s) {
  if (!s) return;
  cudaSetDevice(s->dev);
  if (s->stream) cudaStreamSynchronize(s->stream);
  for (auto& e : s->graphs) cudaGraphExecDestroy(e.exec);
  for (auto* p : {&s->plo, &s->phi})
    for (void* m : p->opened) cudaIpcCloseMemHandle(m);
  for (int i = 0; i < s->nreg; ++i) cudaFree(s->reg[i]);
  cudaFree(s->coef);
  cudaFree(s->kdev);
  cudaFree(s->cot);
  cudaFree(s->flag);
  cudaFree(s->stage_dev);
  cudaFree(s->obs_dev);
  cudaFree(s->obs_w);
  if (s->hflag) cudaFreeHost(s->hflag);
  if (s->obs_host) cudaFreeHost(s->obs_host);
  if (s->own) cudaStreamDestroy(s->own);
  delete s;
}

int hwg_peer_export(hwg_solver* s, hwg_peer_desc* out) {
  return guarded(s, [&]() -> int {
    cudaSetDevice(s->dev);
    std::memset(out, 0, sizeof(*out));
    int rc = ensure_regs(s, 5);
    if (rc) return rc;
    for (int i = 0; i < 5; ++i) {
      out->reg[i] = s->reg[i];
      cudaIpcMemHandle_t h;
      CK(cudaIpcGetMemHandle(&h, s->reg[i]));
      std::memcpy(out->ipc[i], &h, sizeof(h));
    }
    out->flag = s->flag;
    cudaIpcMemHandle_t h;
    CK(cudaIpcGetMemHandle(&h, s->flag));
    std::memcpy(out->ipc[5], &h, sizeof(h));
    out->nrho = s->n;
    out->row_elems = (long long)s->rs;
    out->device = s->dev;
    CK(cudaStreamSynchronize(s->stream));  // registers zeroed before anyone maps them
    return HWG_OK;
  });
}

int hwg_set_peers(hwg_solver* s, const hwg_peer_desc* lower, const hwg_peer_desc* upper,
                  int use_ipc, double timeout_s) {
  return guarded(s, [&]() -> int {
    NvtxRange nvtx_("hwg_set_peers");
    cudaSetDevice(s->dev);
    if (s->ddm) {
      s->err = "hwg_set_peers: fused halo push is implemented for the fp64 / mixed tiers";
      return HWG_EINVAL;
    }
    if ((lower && s->phys_lo) || (upper && s->phys_hi)) {
      s->err = "hwg_set_peers: a neighbour on a physical (excision / scri) end";
      return HWG_EINVAL;
    }
    int rc = ensure_regs(s, 5);
    if (rc) return rc;
    CK(cudaStreamSynchronize(s->stream));
    for (auto* p : {&s->plo, &s->phi}) {
      for (void* m : p->opened) cudaIpcCloseMemHandle(m);
      *p = hwg_solver::Peer{};
    }
    const hwg_peer_desc* ds[2] = {lower, upper};
    hwg_solver::Peer* ps[2] = {&s->plo, &s->phi};
    for (int q = 0; q < 2; ++q) {
      const hwg_peer_desc* d = ds[q];
      if (!d) continue;
      if (d->row_elems != (long long)s->rs) {
        s->err = "hwg_set_peers: neighbour row pitch differs (ntheta must match)";
        return HWG_EINVAL;
      }
      hwg_solver::Peer& p = *ps[q];
      for (int i = 0; i < 6; ++i) {
        void* ptr = i < 5 ? d->reg[i] : d->flag;
        if (use_ipc) {
          cudaIpcMemHandle_t h;
          std::memcpy(&h, d->ipc[i], sizeof(h));
          CK(cudaIpcOpenMemHandle(&ptr, h, cudaIpcMemLazyEnablePeerAccess));
          p.opened.push_back(ptr);
        } else if (d->device != s->dev) {
          cudaError_t e = cudaDeviceEnablePeerAccess(d->device, 0);
          if (e == cudaErrorPeerAccessAlreadyEnabled) cudaGetLastError();
          else CK(e);
        }
        if (i < 5) p.reg[i] = static_cast<double2*>(ptr);
        else p.flag = static_cast<unsigned long long*>(ptr);
      }
      p.n = d->nrho;
      p.on = true;
    }
    s->peer_timeout_ns = (long long)(timeout_s > 0 ? timeout_s * 1e9 : 10e9);
    // counters, epoch and ticket restart at 0; graphs baked the old peer args
    for (auto& e : s->graphs) cudaGraphExecDestroy(e.exec);
    s->graphs.clear();
    CK(cudaMemsetAsync(s->flag + 4, 0, 5 * sizeof(unsigned long long), s->stream));
    CK(cudaStreamSynchronize(s->stream));
    return HWG_OK;
  });
}

int hwg_peer_prime(hwg_solver* s) {
  return guarded(s, [&]() -> int {
    NvtxRange nvtx_("hwg_peer_prime");
    cudaSetDevice(s->dev);
    const int h = halo_rows(s->d.scheme);
    const size_t bytes = (size_t)h * s->rs * sizeof(double2);
    const int c = s->cur;
    if (s->plo.on)
      CK(cudaMemcpyAsync(s->plo.reg[c] + (size_t)(kHalo + s->plo.n) * s->rs, row0(s, c), bytes,
                         cudaMemcpyDefault, s->stream));
    if (s->phi.on)
      CK(cudaMemcpyAsync(s->phi.reg[c] + (size_t)(kHalo - h) * s->rs, row0(s, c) + (size_t)(s->n - h) * s->rs,
                         bytes, cudaMemcpyDefault, s->stream));
    CK(cudaStreamSynchronize(s->stream));
    return HWG_OK;
  });
}

int hwg_set_stream(hwg_solver* s, void* stream, int own) {
  return guarded(s, [&]() -> int {
    s->stream = own ? s->own : static_cast<cudaStream_t>(stream);
    return HWG_OK;
  });
}

int hwg_set_state_dd(hwg_solver* s, const double* u) {
  return guarded(s, [&]() -> int {
    NvtxRange nvtx_("hwg_set_state_dd");
    cudaSetDevice(s->dev);
    int rc = upload_layout(s, u, 2, s->cur);
    if (rc) return rc;
    CK(cudaMemsetAsync(s->flag, 0, 2 * sizeof(unsigned long long), s->stream));
    CK(cudaStreamSynchronize(s->stream));
    return HWG_OK;
  });
}
int hwg_set_state(hwg_solver* s, const double* u) {
  return guarded(s, [&]() -> int {
    NvtxRange nvtx_("hwg_set_state");
    cudaSetDevice(s->dev);
    int rc = upload_layout(s, u, 1, s->cur);
    if (rc) return rc;
    CK(cudaMemsetAsync(s->flag, 0, 2 * sizeof(unsigned long long), s->stream));
    CK(cudaStreamSynchronize(s->stream));
    return HWG_OK;
  });
}
int hwg_get_state_dd(hwg_solver* s, double* u) {
  return guarded(s, [&]() -> int {
    NvtxRange nvtx_("hwg_get_state_dd");
    cudaSetDevice(s->dev);
    return download_layout(s, u, 2, s->cur, true);
  });
}
int hwg_get_state(hwg_solver* s, double* u) {
  return guarded(s, [&]() -> int {
    NvtxRange nvtx_("hwg_get_state");
    cudaSetDevice(s->dev);
    return download_layout(s, u, 1, s->cur, true);
  });
}

int hwg_rhs(hwg_solver* s, double* u, double* du) {
  return guarded(s, [&]() -> int {
    NvtxRange nvtx_("hwg_rhs");
    cudaSetDevice(s->dev);
    return rhs_impl(s, u, du, 1);
  });
}
int hwg_rhs_dd(hwg_solver* s, double* u, double* du) {
  return guarded(s, [&]() -> int {
    NvtxRange nvtx_("hwg_rhs_dd");
    cudaSetDevice(s->dev);
    return rhs_impl(s, u, du, 2);
  });
}

int hwg_launch_stage(hwg_solver* s, int stepper, int stage, double dt_hi, double dt_lo,
                     long long step) {
  return guarded(s, [&]() -> int {
    if (stepper == HWG_SSPRK104) {
      int rc = ensure_regs(s, 5);
      if (rc) return rc;
    }
    const int ns = stepper == HWG_SSPRK33 ? 3 : 10;
    if (stage < 0 || stage >= ns) {
      s->err = "hwg_launch_stage: stage out of range";
      return HWG_EINVAL;
    }
    return do_stage(s, stepper, stage, dt_hi, dt_lo, step);
  });
}

int hwg_launch_steps(hwg_solver* s, int stepper, double dt_hi, double dt_lo,
                     long long step_begin, long long nsteps) {
  return guarded(s, [&]() -> int {
    NvtxRange nvtx_("hwg_launch_steps");
    cudaSetDevice(s->dev);
    return launch_steps_impl(s, stepper, dt_hi, dt_lo, step_begin, nsteps);
  });
}

int hwg_stage_input(const hwg_solver* s, int stepper, int stage, int* reg) {
  return guarded(s, [&]() -> int {
    *reg = stage_input_reg(s, stepper, stage);
    return HWG_OK;
  });
}

int hwg_register_ptr(const hwg_solver* s, int reg, void** row0_ptr, long long* row_elems) {
  return guarded(s, [&]() -> int {
    if (reg < 0 || reg >= s->nreg) return HWG_EINVAL;
    *row0_ptr = row0(s, reg);
    *row_elems = (long long)s->rs;
    return HWG_OK;
  });
}

int hwg_current_register(const hwg_solver* s) { return s->cur; }

int hwg_status(hwg_solver* s, int* blew, long long* step, int clear) {
  return guarded(s, [&]() -> int {
    CK(cudaMemcpyAsync(s->hflag, s->flag, 2 * sizeof(unsigned long long), cudaMemcpyDeviceToHost,
                       s->stream));
    CK(cudaStreamSynchronize(s->stream));
    *blew = s->hflag[0] != 0;
    *step = *blew ? (long long)s->hflag[1] : -1;
    if (clear) {
      CK(cudaMemsetAsync(s->flag, 0, 2 * sizeof(unsigned long long), s->stream));
      CK(cudaMemsetAsync(s->flag + 3, 0, sizeof(unsigned long long), s->stream));
    }
    if (s->hflag[0] & 2ull) {
      s->err = "peer halo wait timed out (a neighbour slab did not run the same stage)";
      return HWG_ERUNTIME;
    }

    return HWG_OK;
  });
}

int hwg_launch_info(const hwg_solver* s, int* blocks, int* threads, int* nranges, int* nchunks,
                    int* pitch) {
  return guarded(s, [&]() -> int {
    *blocks = s->blocks;
    *threads = s->wpb * 32;
    *nranges = s->nranges;
    *nchunks = s->nchunks;
    *pitch = (int)s->rs;
    return HWG_OK;
  });
}

int hwg_synchronize(hwg_solver* s) {
  return guarded(s, [&]() -> int {
    CK(cudaStreamSynchronize(s->stream));
    return HWG_OK;
  });
}

int hwg_set_observers(hwg_solver* s, int kobs, int j0, const double* hw, int jobs,
                      const double* pw) {
  return guarded(s, [&]() -> int {
    if (kobs >= s->nt || j0 + 8 > s->n || jobs >= s->n) {
      s->err = "hwg_set_observers: observer outside this handle's rows";
      return HWG_EINVAL;
    }
    s->kobs = kobs;
    s->j0 = hw ? j0 : -1;
    s->jobs = pw ? jobs : -1;
    std::vector<double> w(32 + s->ntp, 0.0);
    if (hw) std::memcpy(w.data(), hw, 32 * sizeof(double));
    if (pw) std::memcpy(w.data() + 32, pw, s->nt * sizeof(double));
    CK(cudaMemcpy(s->obs_w, w.data(), w.size() * sizeof(double), cudaMemcpyHostToDevice));
    return HWG_OK;
  });
}

int hwg_observe(hwg_solver* s, hwg_observables* out) {
  return guarded(s, [&]() -> int {
    NvtxRange nvtx_("hwg_observe");
    observe_kernel2<<<1, 32, 0, s->stream>>>(row0(s, s->cur), s->rs, s->sblk, s->j0, s->obs_w,
                                              s->kobs, s->jobs, s->phys_hi ? s->n - 1 : -1,
                                              s->obs_w + 32, s->nt, s->obs_dev);
    CK(cudaGetLastError());
    CK(cudaMemcpyAsync(s->obs_host, s->obs_dev, 14 * sizeof(double), cudaMemcpyDeviceToHost,
                       s->stream));
    CK(cudaStreamSynchronize(s->stream));
    const double* o = s->obs_host;
    out->phi[0] = o[0]; out->phi[1] = o[1];
    for (int d = 0; d < 3; ++d) { out->dphi[d][0] = o[2 + 2 * d]; out->dphi[d][1] = o[3 + 2 * d]; }
    out->obs[0] = o[8]; out->obs[1] = o[9];
    out->scri[0] = o[10]; out->scri[1] = o[11];
    out->proj[0] = o[12]; out->proj[1] = o[13];
    return HWG_OK;
  });
}

int hwg_advance(hwg_solver* s, int stepper, double dt_hi, double dt_lo, long long s0,
                long long s1, long long every, hwg_hook_fn hook, void* user,
                hwg_run_stats* stats) {
  return guarded(s, [&]() -> int {
    NvtxRange nvtx_("hwg_advance");
    cudaSetDevice(s->dev);
    s->abort_req = false;
    hwg_run_stats st{0, 0.0, 0, -1};
    if (every < 1) every = 1;
    const long long poll = 256;
    auto t0 = std::chrono::steady_clock::now();
    int rc = HWG_OK;
    long long launched_to = s0;  // steps [s0, launched_to) are queued
    auto check_flag = [&](bool& blown) -> int {
      int b;
      long long bs;
      int r = hwg_status(s, &b, &bs, 0);
      if (r) return r;
      blown = b != 0;
      if (blown) {
        st.blew_up = 1;
        st.blowup_step = bs;
        st.steps_done = bs - s0;
      }
      return HWG_OK;
    };
    {
      // a blow-up flag left by an earlier call: the state is frozen, nothing
      // steps (clear it with hwg_status(clear) or hwg_set_state first)
      bool blown = false;
      if ((rc = check_flag(blown)) == HWG_OK && blown) {
        st.steps_done = 0;
        st.wall_seconds = 0.0;
        if (stats) *stats = st;
        return HWG_OK;
      }
      if (rc) return rc;
    }
    long long q = s0;
    for (;;) {
      const bool hook_now = hook && (q % every == 0 || q == s0 || q == s1);
      if (hook_now || q == s1 || (q - s0) % poll == 0) {
        bool blown = false;
        if ((rc = check_flag(blown))) break;
        if (blown) break;
      }
      if (hook_now) {
        hwg_observables ob;
        if ((rc = hwg_observe(s, &ob))) break;
        DD tau = tau_of(q, dt_hi, dt_lo);
        hook(q, tau.hi, tau.lo, &ob, user);
        if (s->abort_req) break;
      }
      if (q == s1) break;
      // next stop: hook step, poll point or the end
      long long next = std::min(s1, s0 + ((q - s0) / poll + 1) * poll);
      if (hook) next = std::min(next, (q / every + 1) * every);
      if ((rc = launch_steps_impl(s, stepper, dt_hi, dt_lo, q, next - q))) break;
      launched_to = next;
      st.steps_done = launched_to - s0;
      q = next;
    }
    cudaStreamSynchronize(s->stream);
    st.wall_seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    if (stats) *stats = st;
    return rc;
  });
}

int hwg_launch_stage_rows(hwg_solver* s, int stepper, int stage, double dt_hi, double dt_lo,
                          long long step, int row_lo, int row_hi, int part) {
  return guarded(s, [&]() -> int {
    if (s->ddm || s->plo.on || s->phi.on) {
      s->err = "hwg_launch_stage_rows: fast tiers without peer slabs only";
      return HWG_EINVAL;
    }
    const int ns = stepper == HWG_SSPRK33 ? 3 : 10;
    if (stage < 0 || stage >= ns || row_lo < 0 || row_hi > s->n || row_hi - row_lo < 2) {
      s->err = "hwg_launch_stage_rows: stage or row window out of range";
      return HWG_EINVAL;
    }
    if (stepper == HWG_SSPRK104) {
      int rc = ensure_regs(s, 5);
      if (rc) return rc;
    }
    return do_stage_part(s, stepper, stage, dt_hi, dt_lo, step, row_lo, row_hi,
                         (part & HWG_PART_FIRST) != 0, (part & HWG_PART_LAST) != 0);
  });
}

int hwg_peer_stats(hwg_solver* s, long long* spun) {
  return guarded(s, [&]() -> int {
    unsigned long long v = 0;
    CK(cudaMemcpy(&v, s->flag + 8, sizeof(v), cudaMemcpyDeviceToHost));
    *spun = (long long)v;
    return HWG_OK;
  });
}

int hwg_peer_emulate_steps(hwg_solver* const* slabs, int nslabs, int stepper, double dt_hi,
                           double dt_lo, long long step0, long long nsteps, long long skew_ns) {
  if (slabs == nullptr || nslabs < 1 || nslabs > kMaxEmuSlabs || slabs[0] == nullptr)
    return HWG_EINVAL;
  hwg_solver* s0 = slabs[0];
  return guarded(s0, [&]() -> int {
    NvtxRange nvtx_("hwg_peer_emulate_steps");
    cudaSetDevice(s0->dev);
    const int ns = stepper == HWG_SSPRK33 ? 3 : 10;
    for (int k = 0; k < nslabs; ++k) {
      hwg_solver* s = slabs[k];
      if (s == nullptr || s->ddm || s->dev != s0->dev || s->d.scheme != s0->d.scheme ||
          mode_of(s) != mode_of(s0) || nsteps < 0) {
        s0->err = "hwg_peer_emulate_steps: fast-tier slabs of one scheme/precision on one device";
        return HWG_EINVAL;
      }
      if (stepper == HWG_SSPRK104) {
        int rc = ensure_regs(s, 5);
        if (rc) return rc;
      }
    }
    EmuArgs m{};
    m.nslabs = nslabs;
    m.period = 2 * ns;  // the register rotation repeats every two steps
    m.nstages = (int)(nsteps * ns);
    m.skew_ns = skew_ns;
    std::vector<StageArgs> host((size_t)nslabs * m.period);
    int total = 0;
    const DD dt{dt_hi, dt_lo};
    for (int k = 0; k < nslabs; ++k) {
      hwg_solver* s = slabs[k];
      const int rot[5] = {s->cur, s->scr1, s->scr2, s->scr3, s->scr4};
      for (int q = 0; q < m.period; ++q) {
        const int stage = q % ns;
        const Plan p = make_plan(s, stepper, stage, dt);
        int blocks = 0;
        host[(size_t)k * m.period + q] =
            fast_stage_args(s, p, stage, -1, 0, s->n, true, true, &blocks);
        m.epi[q] = p.epi;
        if (p.rot == 1) std::swap(s->cur, s->scr1);
        if (p.rot == 2) std::swap(s->cur, s->scr2);
      }
      s->cur = rot[0]; s->scr1 = rot[1]; s->scr2 = rot[2]; s->scr3 = rot[3]; s->scr4 = rot[4];
      const long long warps = (long long)host[(size_t)k * m.period].nranges * s->nchunks;
      m.s[k].block0 = total;
      m.s[k].blocks = (int)((warps + kWarpsPerBlock - 1) / kWarpsPerBlock);
      total += m.s[k].blocks;
    }
    StageArgs* dargs = nullptr;
    unsigned long long* dbar = nullptr;
    cudaError_t e = cudaDeviceSynchronize();
    if (e == cudaSuccess) e = cudaMalloc(&dargs, host.size() * sizeof(StageArgs));
    if (e == cudaSuccess) e = cudaMalloc(&dbar, nslabs * sizeof(unsigned long long));
    if (e == cudaSuccess)
      e = cudaMemcpy(dargs, host.data(), host.size() * sizeof(StageArgs), cudaMemcpyHostToDevice);
    if (e == cudaSuccess) e = cudaMemset(dbar, 0, nslabs * sizeof(unsigned long long));
    for (int k = 0; k < nslabs && e == cudaSuccess; ++k) {
      m.s[k].args = dargs + (size_t)k * m.period;
      m.s[k].bar = dbar + k;
      set_counter_kernel<<<1, 1, 0, s0->stream>>>(slabs[k]->flag + 2, step0);
      e = cudaGetLastError();
    }
    int capacity = 0;
    if (e == cudaSuccess)
      e = launch_peer_emu(m, s0->d.scheme, mode_of(s0), total, s0->stream, &capacity);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s0->stream);
    if (dargs) cudaFree(dargs);
    if (dbar) cudaFree(dbar);
    if (e != cudaSuccess) {
      s0->err = std::string("hwg_peer_emulate_steps: ") + cudaGetErrorString(e) + " (" +
                std::to_string(total) + " blocks, " + std::to_string(capacity) +
                " co-resident)";
      return HWG_ECUDA;
    }
    // the host's register rotation after nsteps steps
    for (int k = 0; k < nslabs; ++k)
      for (long long q = 0; q < nsteps * ns; ++q) {
        const Plan p = make_plan(slabs[k], stepper, (int)(q % ns), dt);
        if (p.rot == 1) std::swap(slabs[k]->cur, slabs[k]->scr1);
        if (p.rot == 2) std::swap(slabs[k]->cur, slabs[k]->scr2);
      }
    return HWG_OK;
  });
}

int hwg_selftest_division(long long n, unsigned long long seed, long long* mismatches,
                          long long* guard_fails) {
  if (mismatches == nullptr || guard_fails == nullptr || n < 0) return HWG_EINVAL;
  const cudaError_t e = div_selftest(n, seed, mismatches, guard_fails);
  return e == cudaSuccess ? HWG_OK : HWG_ECUDA;
}

int hwg_abort_advance(hwg_solver* s) {
  if (s == nullptr) return HWG_EINVAL;
  s->abort_req = true;
  return HWG_OK;
}

}  // extern "C"
