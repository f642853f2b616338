// Hand-written sm_100a kernels of the dense IRLS alignment (reference
// src/alignment.cpp:367-436, src/warping.cpp:76-114, inc/image.hpp:51-91).
//
// Per IRLS iteration (one launch each, all slots of a batch at once):
//   K1 k_warp_residuals  warp full-res B by T (src/warping.cpp:94-112), stage it
//                        in smem, downsample to the level (src/alignment.cpp:355-363),
//                        residual validity (src/alignment.cpp:206-227) and row-major
//                        compaction of r_I / r_W per tile (systematic-sample ranks).
//   K2 k_tdist           gather the systematic sample (src/alignment.cpp:50-57) and
//                        run the Student-t chain (src/alignment.cpp:61-157,288-320).
//   K3 k_normal_eq       recompute jets (src/alignment.cpp:212-244), robust weights
//                        and the 21+6+1 fp64 sums (src/alignment.cpp:321-335).
//   K4 k_solve           fixed-order reduce, rank test, LDLT, SE(3) update, convergence
//                        (src/alignment.cpp:387-401) — no host round trip.
// Compiled with --fmad=false: mask-deciding arithmetic rounds exactly like the
// reference; reductions use a fixed tree (bit-reproducible run to run).
#include <cuda_runtime.h>
#include <math_constants.h>

#include <cmath>
#include <cstdio>

#include "align_kernels.cuh"

namespace rgbid_b200 {

thread_local long long* g_launch_counter = nullptr;
thread_local Profiler* g_profiler = nullptr;

cudaEvent_t Profiler::get() {
  if (!pool.empty()) {
    cudaEvent_t e = pool.back();
    pool.pop_back();
    return e;
  }
  cudaEvent_t e;
  cudaEventCreate(&e);
  return e;
}

KScope::KScope(const char* n, cudaStream_t s) : name(n), stream(s) {
  if (g_launch_counter) ++*g_launch_counter;
  if (g_profiler && g_profiler->enabled) {
    cudaEvent_t start = g_profiler->get();
    stop = g_profiler->get();
    cudaEventRecord(start, s);
    g_profiler->pending.push_back(KernelRecord{n, start, stop});
  }
}
KScope::~KScope() {
  if (stop) cudaEventRecord(stop, stream);
}

__device__ __forceinline__ bool valid(double v) { return isfinite(v); }

// bilinear — inc/image.hpp:51-62
__device__ __forceinline__ double bilinear(const double* __restrict__ img, int w, int h, double x,
                                           double y) {
  if (!(x >= 0.0 && x <= w - 1.0 && y >= 0.0 && y <= h - 1.0)) return CUDART_NAN;
  const int x0 = (int)floor(x), y0 = (int)floor(y);
  const int x1 = min(x0 + 1, w - 1), y1 = min(y0 + 1, h - 1);
  const double fx = x - x0, fy = y - y0;
  const double v00 = __ldg(img + (size_t)y0 * w + x0), v10 = __ldg(img + (size_t)y0 * w + x1);
  const double v01 = __ldg(img + (size_t)y1 * w + x0), v11 = __ldg(img + (size_t)y1 * w + x1);
  if (!valid(v00) || !valid(v10) || !valid(v01) || !valid(v11)) return CUDART_NAN;
  return (1 - fy) * ((1 - fx) * v00 + fx * v10) + fy * ((1 - fx) * v01 + fx * v11);
}

// one A pixel of inverse_geometric_warp — src/warping.cpp:96-111
__device__ __forceinline__ void warp_px(const WarpMats& m, const double* __restrict__ IB,
                                        const double* __restrict__ WB, int wb, int hb, int x,
                                        int y, double w_a, double& oI, double& oW, double& mx,
                                        double& my) {
  oI = CUDART_NAN;
  oW = CUDART_NAN;
  mx = CUDART_NAN;
  my = CUDART_NAN;
  if (!valid(w_a) || w_a <= 0.0) return;
  const double qx = x / w_a, qy = y / w_a, qz = 1.0 / w_a;
  const double xb0 = red3(m.Rt_BA[0] * qx, m.Rt_BA[1] * qy, m.Rt_BA[2] * qz) + m.tt_BA[0];
  const double xb1 = red3(m.Rt_BA[3] * qx, m.Rt_BA[4] * qy, m.Rt_BA[5] * qz) + m.tt_BA[1];
  const double xb2 = red3(m.Rt_BA[6] * qx, m.Rt_BA[7] * qy, m.Rt_BA[8] * qz) + m.tt_BA[2];
  if (xb2 <= 1e-12) return;
  const double px = xb0 / xb2, py = xb1 / xb2;
  mx = px;
  my = py;
  oI = bilinear(IB, wb, hb, px, py);
  const double w_meas = bilinear(WB, wb, hb, px, py);
  if (!valid(w_meas) || w_meas <= 0.0) return;
  const double rz = red3(m.Rt_AB[6] * px, m.Rt_AB[7] * py, m.Rt_AB[8] * 1.0);
  const double za = rz / w_meas + m.tt_AB[2];
  if (za <= 1e-12) return;
  oW = 1.0 / za;
}

__device__ __forceinline__ double px_or_nan(const double* img, int w, int h, int x, int y) {
  return (x >= 0 && x < w && y >= 0 && y < h) ? __ldg(img + (size_t)y * w + x) : CUDART_NAN;
}

// gradient_at — src/alignment.cpp:165-191
__device__ __forceinline__ bool gradient_at(const double* img, int w, int h, int x, int y,
                                            double& gx, double& gy) {
  const double c = px_or_nan(img, w, h, x, y);
  if (!valid(c)) return false;
  const double l = px_or_nan(img, w, h, x - 1, y), r = px_or_nan(img, w, h, x + 1, y);
  if (valid(l) && valid(r))
    gx = (r - l) / 2.0;
  else if (valid(r))
    gx = r - c;
  else if (valid(l))
    gx = c - l;
  else
    return false;
  const double u = px_or_nan(img, w, h, x, y - 1), d = px_or_nan(img, w, h, x, y + 1);
  if (valid(u) && valid(d))
    gy = (d - u) / 2.0;
  else if (valid(d))
    gy = d - c;
  else if (valid(u))
    gy = c - u;
  else
    return false;
  return true;
}

__device__ __forceinline__ bool gradient_ok(const double* img, int w, int h, int x, int y) {
  if (!valid(px_or_nan(img, w, h, x, y))) return false;
  if (!valid(px_or_nan(img, w, h, x - 1, y)) && !valid(px_or_nan(img, w, h, x + 1, y)))
    return false;
  if (!valid(px_or_nan(img, w, h, x, y - 1)) && !valid(px_or_nan(img, w, h, x, y + 1)))
    return false;
  return true;
}

// 2x2 NaN-aware mean — inc/image.hpp:73-91 (tap order (0,0),(1,0),(0,1),(1,1))
__device__ __forceinline__ double ds4(double a, double b, double c, double d) {
  double sum = 0.0;
  int n = 0;
  if (valid(a)) sum += a, ++n;
  if (valid(b)) sum += b, ++n;
  if (valid(c)) sum += c, ++n;
  if (valid(d)) sum += d, ++n;
  return n > 0 ? sum / n : CUDART_NAN;
}

__device__ __forceinline__ void load_wm(const WarpMats& g, WarpMats& m) {
#pragma unroll
  for (int i = 0; i < 9; ++i) {
    m.Rt_BA[i] = g.Rt_BA[i];
    m.Rt_AB[i] = g.Rt_AB[i];
  }
#pragma unroll
  for (int i = 0; i < 3; ++i) {
    m.tt_BA[i] = g.tt_BA[i];
    m.tt_AB[i] = g.tt_AB[i];
  }
}

// ---------------------------------------------------------------------------
// K1: warp + downsample-to-level + residual validity + per-tile compaction.
template <int L>
__global__ void __launch_bounds__(kTPB) k_warp_residuals(const SlotIO* __restrict__ io,
                                                         const SlotState* __restrict__ st,
                                                         LevelInfo li, int w0, int h0, int phase) {
  const int slot = blockIdx.y;
  if (!slot_active(st[slot], L, phase)) return;
  const SlotIO& o = io[slot];
  const double* WAw = phase ? o.fWA : o.WA[0];
  const double* IAl = phase ? o.fIA : o.IA[L];
  const double* WAl = phase ? o.fWA : o.WA[L];
  WarpMats m;
  load_wm(st[slot].wm, m);

  const int tid = threadIdx.x;
  const int tile = blockIdx.x;
  const int yl = tile / li.nseg, seg = tile - yl * li.nseg;
  const int xl0 = seg * li.tx;
  const int nx = min(li.tx, li.w - xl0);
  double ib = CUDART_NAN, wb = CUDART_NAN, d0, d1;

  if constexpr (L == 0) {
    if (tid < nx) {
      const int x = xl0 + tid;
      warp_px(m, o.IB, o.WB, w0, h0, x, yl, __ldg(WAw + (size_t)yl * w0 + x), ib, wb, d0, d1);
    }
  } else {
    __shared__ double sI[2048], sW[2048];
    int cw = nx << L, ch = 1 << L;
    const int npx = cw * ch;
    for (int k = tid; k < npx; k += kTPB) {
      const int r = k / cw, c = k - r * cw;
      const int x = (xl0 << L) + c, y = (yl << L) + r;
      double vi, vw;
      warp_px(m, o.IB, o.WB, w0, h0, x, y, __ldg(WAw + (size_t)y * w0 + x), vi, vw, d0, d1);
      sI[k] = vi;
      sW[k] = vw;
    }
    __syncthreads();
#pragma unroll
    for (int s = 0; s < L; ++s) {
      const int ow = cw >> 1, oh = ch >> 1, nout = ow * oh;
      double oi[2], owv[2];
#pragma unroll
      for (int q = 0; q < 2; ++q) {
        const int k = tid + q * kTPB;
        if (k < nout) {
          const int r = k / ow, c = k - r * ow;
          const int i0 = (2 * r) * cw + 2 * c, i1 = i0 + cw;
          oi[q] = ds4(sI[i0], sI[i0 + 1], sI[i1], sI[i1 + 1]);
          owv[q] = ds4(sW[i0], sW[i0 + 1], sW[i1], sW[i1 + 1]);
        }
      }
      __syncthreads();
#pragma unroll
      for (int q = 0; q < 2; ++q) {
        const int k = tid + q * kTPB;
        if (k < nout) {
          sI[k] = oi[q];
          sW[k] = owv[q];
        }
      }
      __syncthreads();
      cw = ow;
      ch = oh;
    }
    if (tid < nx) {
      ib = sI[tid];
      wb = sW[tid];
    }
  }

  bool jet = false, dep = false;
  double rI = 0.0, rW = 0.0;
  if (tid < nx) {
    const int xl = xl0 + tid;
    const size_t idx = (size_t)yl * li.w + xl;
    o.ib[idx] = ib;
    o.wb[idx] = wb;
    const double w_a = __ldg(WAl + idx), i_a = __ldg(IAl + idx);
    if (valid(w_a) && w_a > 0.0 && valid(i_a) && valid(ib) && gradient_ok(IAl, li.w, li.h, xl, yl)) {
      jet = true;
      rI = ib - i_a;
      if (valid(wb) && wb > 0.0 && gradient_ok(WAl, li.w, li.h, xl, yl)) {
        dep = true;
        rW = wb - w_a;
      }
    }
  }
  // block compaction in row-major order (tid order == x order)
  __shared__ int wcnt[2][kTPB / 32];
  const int lane = tid & 31, wid = tid >> 5;
  const unsigned bj = __ballot_sync(0xffffffffu, jet), bd = __ballot_sync(0xffffffffu, dep);
  if (lane == 0) {
    wcnt[0][wid] = __popc(bj);
    wcnt[1][wid] = __popc(bd);
  }
  __syncthreads();
  int offI = 0, offW = 0, totI = 0, totW = 0;
#pragma unroll
  for (int k = 0; k < kTPB / 32; ++k) {
    if (k < wid) {
      offI += wcnt[0][k];
      offW += wcnt[1][k];
    }
    totI += wcnt[0][k];
    totW += wcnt[1][k];
  }
  const unsigned lt = (1u << lane) - 1u;
  const size_t base = (size_t)yl * li.w + xl0;
  if (jet) o.resI[base + offI + __popc(bj & lt)] = rI;
  if (dep) o.resW[base + offW + __popc(bd & lt)] = rW;
  if (tid == 0) {
    o.cntI[tile] = totI;
    o.cntW[tile] = totW;
  }
}

void launch_warp_residuals(const AlignLaunch& a, const LevelInfo& li, int phase, cudaStream_t s) {
  KScope ks_("warp_residuals", s);
  dim3 grid(li.ntiles, a.nslots);
  switch (li.level) {
    case 0: k_warp_residuals<0><<<grid, kTPB, 0, s>>>(a.io, a.st, li, a.w0, a.h0, phase); break;
    case 1: k_warp_residuals<1><<<grid, kTPB, 0, s>>>(a.io, a.st, li, a.w0, a.h0, phase); break;
    case 2: k_warp_residuals<2><<<grid, kTPB, 0, s>>>(a.io, a.st, li, a.w0, a.h0, phase); break;
    case 3: k_warp_residuals<3><<<grid, kTPB, 0, s>>>(a.io, a.st, li, a.w0, a.h0, phase); break;
    case 4: k_warp_residuals<4><<<grid, kTPB, 0, s>>>(a.io, a.st, li, a.w0, a.h0, phase); break;
    case 5: k_warp_residuals<5><<<grid, kTPB, 0, s>>>(a.io, a.st, li, a.w0, a.h0, phase); break;
    default: return;
  }
}

// ---------------------------------------------------------------------------
// Block-wide fixed-order reductions (every thread receives the bit-identical total).
template <int NV, int NT>
__device__ __forceinline__ void block_allsum(double (&v)[NV], double* scratch) {
  constexpr int NW = NT / 32;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
#pragma unroll
  for (int off = 16; off > 0; off >>= 1)
#pragma unroll
    for (int i = 0; i < NV; ++i) v[i] += __shfl_xor_sync(0xffffffffu, v[i], off);
  if (lane == 0)
#pragma unroll
    for (int i = 0; i < NV; ++i) scratch[wid * NV + i] = v[i];
  __syncthreads();
#pragma unroll
  for (int i = 0; i < NV; ++i) v[i] = lane < NW ? scratch[lane * NV + i] : 0.0;
#pragma unroll
  for (int off = 16; off > 0; off >>= 1)
#pragma unroll
    for (int i = 0; i < NV; ++i) v[i] += __shfl_xor_sync(0xffffffffu, v[i], off);
  __syncthreads();
}

struct TD {
  double mu, sigma, nu;
};

__device__ __forceinline__ double t_weight(double x, double nu) { return (nu + 1.0) / (nu + x * x); }

// estimate_location_scale on the (already sampled) smem vector — src/alignment.cpp:61-101
template <int NT>
__device__ TD loc_scale(const double* smp, int m, double nu, double* scratch) {
  TD p{0.0, 1.0, nu};
  if (m == 0) return p;
  const int tid = threadIdx.x;
  double a1[1] = {0.0};
  for (int i = tid; i < m; i += NT) a1[0] += smp[i];
  block_allsum<1, NT>(a1, scratch);
  double mu = a1[0] / (double)m;
  a1[0] = 0.0;
  for (int i = tid; i < m; i += NT) {
    const double d = smp[i] - mu;
    a1[0] += d * d;
  }
  block_allsum<1, NT>(a1, scratch);
  double sigma = sqrt(a1[0] / (double)m);
  if (sigma < 1e-8) return TD{mu, 1e-8, nu};
  for (int it = 0; it < 50; ++it) {
    double a2[2] = {0.0, 0.0};
    for (int i = tid; i < m; i += NT) {
      const double v = smp[i];
      const double w = t_weight((v - mu) / sigma, nu);
      a2[0] += w;
      a2[1] += w * v;
    }
    block_allsum<2, NT>(a2, scratch);
    const double mu_new = a2[1] / a2[0];
    a1[0] = 0.0;
    for (int i = tid; i < m; i += NT) {
      const double v = smp[i];
      const double w = t_weight((v - mu_new) / sigma, nu);
      a1[0] += w * (v - mu_new) * (v - mu_new);
    }
    block_allsum<1, NT>(a1, scratch);
    const double sigma_new = dmax_std(1e-8, sqrt(a1[0] / (double)m));
    const double rel = fabs(sigma_new - sigma) / sigma;
    mu = mu_new;
    sigma = sigma_new;
    if (rel < 1e-4) break;
  }
  return TD{mu, dmax_std(sigma, 1e-8), nu};
}

// digamma — src/alignment.cpp:32-43
__device__ __forceinline__ double digamma_d(double x) {
  double result = 0.0;
  while (x < 6.0) {
    result -= 1.0 / x;
    x += 1.0;
  }
  const double inv = 1.0 / x;
  const double inv2 = inv * inv;
  result += log(x) - 0.5 * inv - inv2 * (1.0 / 12.0 - inv2 * (1.0 / 120.0 - inv2 / 252.0));
  return result;
}

// stationarity of solve_nu — src/alignment.cpp:132-141.  The nu-only part C is
// hoisted; each per-sample term (C + log w) - w is bit-identical to the reference's.
template <int NT>
__device__ double stationarity(const double* smp, int m, double mu, double sigma, double nu,
                               double* scratch) {
  const double C = (((-digamma_d(nu / 2.0) + log(nu / 2.0)) + digamma_d((nu + 1.0) / 2.0)) -
                    log((nu + 1.0) / 2.0)) + 1.0;
  double a[1] = {0.0};
  for (int i = threadIdx.x; i < m; i += NT) {
    const double w = t_weight((smp[i] - mu) / sigma, nu);
    a[0] += (C + log(w)) - w;
  }
  block_allsum<1, NT>(a, scratch);
  return a[0] / (double)m;
}

// solve_nu — src/alignment.cpp:131-157
template <int NT>
__device__ double solve_nu(const double* smp, int m, double mu, double sigma, double* scratch) {
  double lo = 2.0, hi = 10.0;
  double flo = stationarity<NT>(smp, m, mu, sigma, lo, scratch);
  const double fhi = stationarity<NT>(smp, m, mu, sigma, hi, scratch);
  if (flo * fhi > 0.0) return fhi > 0.0 ? hi : lo;
  for (int it = 0; it < 30; ++it) {
    const double mid = 0.5 * (lo + hi);
    const double fmid = stationarity<NT>(smp, m, mu, sigma, mid, scratch);
    if (flo * fmid <= 0.0) {
      hi = mid;
    } else {
      lo = mid;
      flo = fmid;
    }
  }
  return 0.5 * (lo + hi);
}

// estimate_nu — src/alignment.cpp:109-127
template <int NT>
__device__ double estimate_nu(const double* smp, int m, double mu, double sigma, double* scratch) {
  if (m == 0 || sigma <= 0.0) return 5.0;
  double nu = solve_nu<NT>(smp, m, mu, sigma, scratch);
  for (int it = 0; it < 2 && nu < 9.99; ++it) {
    const TD refit = loc_scale<NT>(smp, m, nu, scratch);
    if (refit.sigma <= 0.0) break;
    const double nu_new = solve_nu<NT>(smp, m, refit.mu, refit.sigma, scratch);
    if (fabs(nu_new - nu) < 1e-3) {
      nu = nu_new;
      break;
    }
    nu = nu_new;
  }
  return nu;
}

__global__ void k_tdist(const SlotIO* __restrict__ io, SlotState* __restrict__ st, LevelInfo li,
                        int phase);

int init_kernel_attributes() {
  // sample (19200 doubles) + tile offsets; static smem of k_tdist is small
  const cudaError_t e =
      cudaFuncSetAttribute(k_tdist, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  cudaGetLastError();  // do not leave a sticky error for the next launch check
  return e == cudaSuccess ? 0 : 1;
}

int tdist_smem_bytes(int ntiles) {
  return kMaxSample * 8 + (ntiles + 1) * 4 + 64 * 8 + 16;
}

// K2: systematic sample + Student-t chain for one (slot, residual type).
__global__ void __launch_bounds__(kTdistThreads) k_tdist(const SlotIO* __restrict__ io,
                                                         SlotState* __restrict__ st, LevelInfo li,
                                                         int phase) {
  constexpr int NT = kTdistThreads;
  const int type = blockIdx.x, slot = blockIdx.y;
  SlotState& S = st[slot];
  if (!slot_active(S, li.level, phase)) return;
  const SlotIO& o = io[slot];
  const int* cnt = type ? o.cntW : o.cntI;
  const double* res = type ? o.resW : o.resI;
  extern __shared__ double dsm[];
  double* smp = dsm;
  double* scratch = dsm + kMaxSample;                    // 64 doubles
  int* offs = reinterpret_cast<int*>(scratch + 64);      // ntiles + 1
  __shared__ int wsum[NT / 32];
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int nt = li.ntiles;

  // exclusive scan of per-tile counts (contiguous chunk per thread)
  const int per = (nt + NT - 1) / NT;
  const int b0 = min(nt, tid * per), b1 = min(nt, b0 + per);
  int local = 0;
  for (int i = b0; i < b1; ++i) local += cnt[i];
  int incl = local;
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {
    const int v = __shfl_up_sync(0xffffffffu, incl, off);
    if (lane >= off) incl += v;
  }
  if (lane == 31) wsum[wid] = incl;
  __syncthreads();
  int woff = 0;
  for (int k = 0; k < wid; ++k) woff += wsum[k];
  int run = woff + incl - local;
  for (int i = b0; i < b1; ++i) {
    offs[i] = run;
    run += cnt[i];
  }
  int total = 0;
  for (int k = 0; k < NT / 32; ++k) total += wsum[k];
  if (tid == 0) offs[nt] = total;
  __syncthreads();

  const long long n = total;
  const long long stride = n <= kMaxSample ? 1 : (n + kMaxSample - 1) / kMaxSample;
  const int m = n == 0 ? 0 : (int)((n - 1) / stride + 1);
  for (int s = tid; s < m; s += NT) {
    const long long g = (long long)s * stride;
    int lo = 0, hi = nt - 1;
    while (lo < hi) {  // last tile with offs[t] <= g
      const int mid = (lo + hi + 1) >> 1;
      if (offs[mid] <= g)
        lo = mid;
      else
        hi = mid - 1;
    }
    const int yl = lo / li.nseg, seg = lo - yl * li.nseg;
    smp[s] = res[(size_t)yl * li.w + (size_t)seg * li.tx + (size_t)(g - offs[lo])];
  }
  __syncthreads();

  // build_system's Student-t part — src/alignment.cpp:305-317
  TD t = loc_scale<NT>(smp, m, 5.0, scratch);
  t.sigma = dmax_std(t.sigma, 1e-8);
  t.nu = estimate_nu<NT>(smp, m, t.mu, t.sigma, scratch);
  if (t.nu < 4.99) {
    const TD r = loc_scale<NT>(smp, m, t.nu, scratch);
    if (r.sigma > 0.0) {
      t.mu = r.mu;
      t.sigma = dmax_std(r.sigma, 1e-8);
    }
  }
  if (tid == 0) {
    rgbid_tdist out{t.mu, t.sigma, t.nu};
    if (type == 0) {
      S.tI = out;
      S.nI = n;
    } else {
      S.tW = out;
      S.nW = n;
    }
  }
}

void launch_tdist(const AlignLaunch& a, const LevelInfo& li, int phase, cudaStream_t s) {
  const int smem = tdist_smem_bytes(li.ntiles);  // <= 200 KB for ntiles <= 11000
  KScope ks_("tdist", s);
  k_tdist<<<dim3(2, a.nslots), kTdistThreads, smem, s>>>(a.io, a.st, li, phase);
}

// ---------------------------------------------------------------------------
// K3: jets + robust weights + 28 fp64 sums per tile.
struct Jet {
  double rI, rW, JI[6], JW[6], lambda;
  bool depth;
};

// residuals_and_jacobians for one pixel — src/alignment.cpp:206-246
__device__ __forceinline__ bool jet_at(const double* IA, const double* WA, double i_b, double w_b,
                                       int w, int h, int x, int y, const LevelInfo& li,
                                       double lambda_n_min, Jet& j) {
  const size_t i = (size_t)y * w + x;
  const double w_a = __ldg(WA + i), i_a = __ldg(IA + i);
  if (!valid(w_a) || w_a <= 0.0 || !valid(i_a) || !valid(i_b)) return false;
  double gix, giy;
  if (!gradient_at(IA, w, h, x, y, gix, giy)) return false;
  // A = K - p e_z^T ; X_A = K^-1 p / w_a ; M = [I | -[X_A]x]
  const double px = x, py = y;
  double A[3][3] = {{li.fx, 0.0, li.cx - px}, {0.0, li.fy, li.cy - py}, {0.0, 0.0, 1.0 - 1.0}};
  const double* Ki = li.Kinv;
  const double X0 = red3(Ki[0] * px, Ki[1] * py, Ki[2] * 1.0) / w_a;
  const double X1 = red3(Ki[3] * px, Ki[4] * py, Ki[5] * 1.0) / w_a;
  const double X2 = red3(Ki[6] * px, Ki[7] * py, Ki[8] * 1.0) / w_a;
  const double M[3][6] = {{1.0, 0.0, 0.0, -0.0, X2, -X1},
                          {0.0, 1.0, 0.0, -X2, -0.0, X0},
                          {0.0, 0.0, 1.0, X1, -X0, -0.0}};
  j.rI = i_b - i_a;
  j.rW = 0.0;
  j.lambda = 1.0;
  j.depth = false;
  {
    const double s0 = w_a * gix, s1 = w_a * giy, s2 = w_a * 0.0;
    double u[3];
#pragma unroll
    for (int c = 0; c < 3; ++c) u[c] = red3(s0 * A[0][c], s1 * A[1][c], s2 * A[2][c]);
#pragma unroll
    for (int c = 0; c < 6; ++c) j.JI[c] = red3(u[0] * M[0][c], u[1] * M[1][c], u[2] * M[2][c]);
  }
  double gwx, gwy;
  if (!(valid(w_b) && w_b > 0.0 && gradient_at(WA, w, h, x, y, gwx, gwy))) return true;
  j.depth = true;
  j.rW = w_b - w_a;
  double gA[3], s2v[3];
#pragma unroll
  for (int c = 0; c < 3; ++c) gA[c] = red3(gwx * A[0][c], gwy * A[1][c], 0.0 * A[2][c]);
  s2v[0] = w_a * (gA[0] + w_b * 0.0);
  s2v[1] = w_a * (gA[1] + w_b * 0.0);
  s2v[2] = w_a * (gA[2] + w_b * 1.0);
#pragma unroll
  for (int c = 0; c < 6; ++c) j.JW[c] = red3(s2v[0] * M[0][c], s2v[1] * M[1][c], s2v[2] * M[2][c]);
  double n0 = gA[0] / w_a + 0.0, n1 = gA[1] / w_a + 0.0, n2 = gA[2] / w_a + 1.0;
  const double nn = sqrt(red3(n0 * n0, n1 * n1, n2 * n2));
  if (!(nn < 1e-12)) {
    n0 /= nn;
    n1 /= nn;
    n2 /= nn;
    if (n2 < 0) {
      n0 = -n0;
      n1 = -n1;
      n2 = -n2;
    }
    double r0 = red3(Ki[0] * px, Ki[1] * py, Ki[2] * 1.0);  // ray = K^-1 p
    double r1 = red3(Ki[3] * px, Ki[4] * py, Ki[5] * 1.0);
    double r2 = red3(Ki[6] * px, Ki[7] * py, Ki[8] * 1.0);
    const double sq = red3(r0 * r0, r1 * r1, r2 * r2);
    if (sq > 0.0) {
      const double sn = sqrt(sq);
      r0 /= sn;
      r1 /= sn;
      r2 /= sn;
    }
    j.lambda = dmax_std(lambda_n_min, red3(n0 * r0, n1 * r1, n2 * r2));
  }
  return true;
}

template <int NT>
__device__ __forceinline__ void block_sum_to(double (&v)[kNPart], double* out, double* scratch) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
#pragma unroll
  for (int off = 16; off > 0; off >>= 1)
#pragma unroll
    for (int i = 0; i < kNPart; ++i) v[i] += __shfl_down_sync(0xffffffffu, v[i], off);
  if (lane == 0)
#pragma unroll
    for (int i = 0; i < kNPart; ++i) scratch[wid * kNPart + i] = v[i];
  __syncthreads();
  if (threadIdx.x < kNPart) {
    double s = 0.0;
    for (int k = 0; k < NT / 32; ++k) s += scratch[k * kNPart + threadIdx.x];
    out[threadIdx.x] = s;
  }
}

__global__ void __launch_bounds__(kTPB) k_normal_eq(const SlotIO* __restrict__ io,
                                                    const SlotState* __restrict__ st, LevelInfo li,
                                                    int phase, double lambda_n_min) {
  const int slot = blockIdx.y;
  const SlotState& S = st[slot];
  if (!slot_active(S, li.level, phase)) return;
  const SlotIO& o = io[slot];
  const double* IAl = phase ? o.fIA : o.IA[li.level];
  const double* WAl = phase ? o.fWA : o.WA[li.level];
  __shared__ double scratch[(kTPB / 32) * kNPart];
  const double muI = S.tI.mu, sgI = S.tI.sigma, nuI = dmax_std(S.tI.nu, S.tW.nu);
  const double muW = S.tW.mu, sgW = S.tW.sigma, nuW = S.tW.nu;
  const double s2i = sgI * sgI, s2w = sgW * sgW;
  double acc[kNPart];
#pragma unroll
  for (int i = 0; i < kNPart; ++i) acc[i] = 0.0;
  const long long k = (long long)blockIdx.x * kTPB + threadIdx.x;
  const long long N = (long long)li.w * li.h;
  if (k < N) {
    const int y = (int)(k / li.w), x = (int)(k - (long long)y * li.w);
    Jet j;
    if (jet_at(IAl, WAl, o.ib[k], o.wb[k], li.w, li.h, x, y, li, lambda_n_min, j)) {
      const double wi = t_weight((j.rI - muI) / sgI, nuI) / s2i;
      int q = 0;
#pragma unroll
      for (int a = 0; a < 6; ++a) {
        const double va = wi * j.JI[a];
#pragma unroll
        for (int c = 0; c <= a; ++c) acc[q++] += va * j.JI[c];
      }
#pragma unroll
      for (int a = 0; a < 6; ++a) acc[21 + a] += (wi * j.JI[a]) * j.rI;
      acc[27] += wi * j.rI * j.rI;
      if (j.depth) {
        const double ww = j.lambda * t_weight((j.rW - muW) / sgW, nuW) / s2w;
        q = 0;
#pragma unroll
        for (int a = 0; a < 6; ++a) {
          const double va = ww * j.JW[a];
#pragma unroll
          for (int c = 0; c <= a; ++c) acc[q++] += va * j.JW[c];
        }
#pragma unroll
        for (int a = 0; a < 6; ++a) acc[21 + a] += (ww * j.JW[a]) * j.rW;
        acc[27] += ww * j.rW * j.rW;
      }
    }
  }
  block_sum_to<kTPB>(acc, o.part + (size_t)blockIdx.x * kNPart, scratch);
}

void launch_normal_equations(const AlignLaunch& a, const LevelInfo& li, int phase, cudaStream_t s) {
  KScope ks_("normal_eq", s);
  k_normal_eq<<<dim3(li.ntiles3, a.nslots), kTPB, 0, s>>>(a.io, a.st, li, phase, a.lambda_n_min);
}

// fixed-order reduction of the per-tile partials into H (full, mirrored), b, cost
__device__ void reduce_partials(const double* part, int ntiles, double* H, double* b, double* cost,
                                double* sh /*[kTPB/32 * kNPart]*/) {
  double acc[kNPart];
#pragma unroll
  for (int i = 0; i < kNPart; ++i) acc[i] = 0.0;
  for (int t = threadIdx.x; t < ntiles; t += kTPB)
#pragma unroll
    for (int i = 0; i < kNPart; ++i) acc[i] += part[(size_t)t * kNPart + i];
  __shared__ double tot[kNPart];
  block_sum_to<kTPB>(acc, tot, sh);
  __syncthreads();
  if (threadIdx.x == 0) {
    int q = 0;
    for (int r = 0; r < 6; ++r)
      for (int c = 0; c <= r; ++c) {
        H[r * 6 + c] = tot[q];
        H[c * 6 + r] = tot[q];
        ++q;
      }
    for (int r = 0; r < 6; ++r) b[r] = -tot[21 + r];
    *cost = tot[27];
  }
}

// K4: solve + pose update + convergence — src/alignment.cpp:387-401
__global__ void __launch_bounds__(kTPB) k_solve(const SlotIO* __restrict__ io,
                                                SlotState* __restrict__ st,
                                                rgbid_iter_trace* __restrict__ trace, LevelInfo li,
                                                int w0, int h0, double fx0, double fy0, double cx0,
                                                double cy0, double eps) {
  const int slot = blockIdx.x;
  SlotState& S = st[slot];
  if (!slot_active(S, li.level, 0)) return;
  if (S.nI < 6) {  // jets.size() < 6 -> DegenerateAlignmentError(zero spectrum)
    if (threadIdx.x == 0) {
      S.status = RGBID_E_DEGENERATE;
      for (int i = 0; i < 36; ++i) S.H[i] = 0.0;
    }
    return;
  }
  __shared__ double sh[(kTPB / 32) * kNPart];
  __shared__ double H[36], b[6], cost;
  reduce_partials(io[slot].part, li.ntiles3, H, b, &cost, sh);
  if (threadIdx.x != 0) return;
  for (int i = 0; i < 36; ++i) S.H[i] = H[i];
  if (rank_deficient6(H)) {
    S.status = RGBID_E_DEGENERATE;
    return;
  }
  double xi[6];
  ldlt_solve6(H, b, xi);
  const PoseD T = pose_update(xi, pose_from(S.R, S.t));
  pose_to(T, S.R, S.t);
  S.wm = warp_mats(T, fx0, fy0, cx0, cy0);
  const int L = li.level;
  S.iters[L] += 1;
  S.cost[L] = cost;
  S.total_iters += 1;
  rgbid_tdist tI = S.tI;
  tI.nu = dmax_std(S.tI.nu, S.tW.nu);
  if (L == 0) {
    S.finI = tI;
    S.finW = S.tW;
  }
  if (trace && slot == 0 && S.trace_n < kTraceMax) {
    rgbid_iter_trace& e = trace[S.trace_n++];
    e.level = L;
    e.iter = S.iters[L] - 1;
    e.n_jets = S.nI;
    e.n_depth = S.nW;
    e.tI = tI;
    e.tW = S.tW;
    for (int i = 0; i < 36; ++i) e.H[i] = H[i];
    for (int i = 0; i < 6; ++i) {
      e.b[i] = b[i];
      e.xi[i] = xi[i];
    }
    e.cost = cost;
    pose_to(T, e.T_after.R, e.T_after.t);
  }
  const double xn = sqrt(red3(xi[0] * xi[0], xi[1] * xi[1], xi[2] * xi[2]) +
                         red3(xi[3] * xi[3], xi[4] * xi[4], xi[5] * xi[5]));
  if (xn < eps) S.done_level = L;
  (void)w0;
  (void)h0;
}

// K5: filtered-Hessian covariance — src/alignment.cpp:422-435
__global__ void __launch_bounds__(kTPB) k_covariance(const SlotIO* __restrict__ io,
                                                     SlotState* __restrict__ st, int ntiles3) {
  const int slot = blockIdx.x;
  SlotState& S = st[slot];
  if (S.status != RGBID_OK) return;
  if (S.nI < 6) {
    if (threadIdx.x < 36) S.cov[threadIdx.x] = (threadIdx.x % 7 == 0) ? 1e6 : 0.0;
    if (threadIdx.x == 0) S.cov_degenerate = 1;
    return;
  }
  __shared__ double sh[(kTPB / 32) * kNPart];
  __shared__ double H[36], b[6], cost;
  reduce_partials(io[slot].part, ntiles3, H, b, &cost, sh);
  if (threadIdx.x != 0) return;
  double Hs[36], inv[36];
  for (int r = 0; r < 6; ++r)
    for (int c = 0; c < 6; ++c) Hs[r * 6 + c] = (H[r * 6 + c] + H[c * 6 + r]) / 2.0;
  if (rank_deficient6(Hs)) {
    for (int i = 0; i < 36; ++i) S.cov[i] = (i % 7 == 0) ? 1e6 : 0.0;
    S.cov_degenerate = 1;
    return;
  }
  lu_inverse6(Hs, inv);
  for (int r = 0; r < 6; ++r)
    for (int c = 0; c < 6; ++c) S.cov[r * 6 + c] = (inv[r * 6 + c] + inv[c * 6 + r]) / 2.0;
  S.cov_degenerate = 0;
}

void launch_covariance(const AlignLaunch& a, const LevelInfo& li, cudaStream_t s) {
  KScope ks_("covariance", s);
  k_covariance<<<a.nslots, kTPB, 0, s>>>(a.io, a.st, li.ntiles3);
}

void launch_solve(const AlignLaunch& a, const LevelInfo& li, const LevelInfo& li0, cudaStream_t s) {
  KScope ks_("solve", s);
  k_solve<<<a.nslots, kTPB, 0, s>>>(a.io, a.st, a.trace, li, a.w0, a.h0, li0.fx, li0.fy, li0.cx,
                                    li0.cy, a.eps);
}

// ---------------------------------------------------------------------------
// pyramid level: downsample2 of I and W — inc/image.hpp:73-91
__global__ void k_downsample2(const double* __restrict__ I, const double* __restrict__ W, int w,
                              int h, double* __restrict__ oI, double* __restrict__ oW) {
  const int ow = w / 2, oh = h / 2;
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= ow * oh) return;
  const int y = k / ow, x = k - y * ow;
  const size_t i0 = (size_t)(2 * y) * w + 2 * x, i1 = i0 + w;
  if (I) oI[k] = ds4(I[i0], I[i0 + 1], I[i1], I[i1 + 1]);
  oW[k] = ds4(W[i0], W[i0 + 1], W[i1], W[i1 + 1]);
}

void launch_downsample2(const double* I, const double* W, int w, int h, double* oI, double* oW,
                        cudaStream_t s) {
  const int n = (w / 2) * (h / 2);
  if (n <= 0) return;
  KScope ks_("pyramid_downsample2", s);
  k_downsample2<<<(n + 255) / 256, 256, 0, s>>>(I, W, w, h, oI, oW);
}

// bilateral_filter — src/alignment.cpp:252-277
__device__ __forceinline__ double bilateral_px(const double* img, int w, int h, int x, int y,
                                               double inv2ss, double inv2sr) {
  const double c = img[(size_t)y * w + x];
  if (!valid(c)) return CUDART_NAN;
  double wsum = 0.0, vsum = 0.0;
  for (int dy = -2; dy <= 2; ++dy)
    for (int dx = -2; dx <= 2; ++dx) {
      const int sx = x + dx, sy = y + dy;
      if (!(sx >= 0 && sx < w && sy >= 0 && sy < h)) continue;
      const double v = img[(size_t)sy * w + sx];
      if (!valid(v)) continue;
      const double wt = exp(-(dx * dx + dy * dy) * inv2ss - (v - c) * (v - c) * inv2sr);
      wsum += wt;
      vsum += wt * v;
    }
  return vsum / wsum;
}

__global__ void k_bilateral(const double* __restrict__ img, int w, int h, double inv2ss,
                            double inv2sr, double* __restrict__ out) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= w * h) return;
  const int y = k / w, x = k - y * w;
  out[k] = bilateral_px(img, w, h, x, y, inv2ss, inv2sr);
}

void launch_bilateral(const double* img, int w, int h, double ss, double sr, double* out,
                      cudaStream_t s) {
  const double inv2ss = 1.0 / (2.0 * ss * ss), inv2sr = 1.0 / (2.0 * sr * sr);
  KScope ks_("bilateral", s);
  k_bilateral<<<(w * h + 255) / 256, 256, 0, s>>>(img, w, h, inv2ss, inv2sr, out);
}

// both filtered maps of every active slot (covariance pass input)
__global__ void k_bilateral_slots(const SlotIO* __restrict__ io, const SlotState* __restrict__ st,
                                  int w, int h, double inv2ss, double inv2sr_i, double inv2sr_w) {
  const int slot = blockIdx.y;
  if (st[slot].status != RGBID_OK) return;
  const SlotIO& o = io[slot];
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= w * h) return;
  const int y = k / w, x = k - y * w;
  o.fIA[k] = bilateral_px(o.IA[0], w, h, x, y, inv2ss, inv2sr_i);
  o.fWA[k] = bilateral_px(o.WA[0], w, h, x, y, inv2ss, inv2sr_w);
}

void launch_bilateral_pair(const AlignLaunch& a, double ss, double sr_i, double sr_w,
                           cudaStream_t s) {
  const double inv2ss = 1.0 / (2.0 * ss * ss);
  const double ii = 1.0 / (2.0 * sr_i * sr_i), iw = 1.0 / (2.0 * sr_w * sr_w);
  const int n = a.w0 * a.h0;
  KScope ks_("bilateral_slots", s);
  k_bilateral_slots<<<dim3((n + 255) / 256, a.nslots), 256, 0, s>>>(a.io, a.st, a.w0, a.h0,
                                                                     inv2ss, ii, iw);
}

// inverse_geometric_warp producing all four WarpedFrame maps (drop-in + tests)
__global__ void k_warp_maps(const double* __restrict__ IB, const double* __restrict__ WB, int wb,
                            int hb, const double* __restrict__ WA, int w, int h, WarpMats m,
                            double* oI, double* oW, double* omx, double* omy) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= w * h) return;
  const int y = k / w, x = k - y * w;
  double a, b, c, d;
  warp_px(m, IB, WB, wb, hb, x, y, WA[k], a, b, c, d);
  if (oI) oI[k] = a;
  if (oW) oW[k] = b;
  if (omx) omx[k] = c;
  if (omy) omy[k] = d;
}

void launch_warp_maps(const double* IB, const double* WB, int wb, int hb, const double* WA, int w,
                      int h, const WarpMats& m, double* oI, double* oW, double* omx, double* omy,
                      cudaStream_t s) {
  KScope ks_("warp_maps", s);
  k_warp_maps<<<(w * h + 255) / 256, 256, 0, s>>>(IB, WB, wb, hb, WA, w, h, m, oI, oW, omx, omy);
}

}  // namespace rgbid_b200
