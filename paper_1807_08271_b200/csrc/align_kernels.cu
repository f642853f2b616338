// Hand-written sm_100a kernels of the dense IRLS alignment (reference
// src/alignment.cpp:367-436, src/warping.cpp:76-114, inc/image.hpp:51-91).
//
// Per IRLS iteration (one launch each, all slots of a batch at once):
//   K1  k_warp_residuals(_l0)  warp full-res B by T (src/warping.cpp:94-112),
//                        downsample to the level (src/alignment.cpp:355-363),
//                        store r_I = i_b - i_a and w_b, residual validity
//                        (src/alignment.cpp:206-227) as row-major per-tile ballots.
//   K2a k_gather         the systematic sample (src/alignment.cpp:50-57) from the
//                        ballots, compacted in global memory (batches).
//   K2b k_tdist<NT>      the Student-t chain (src/alignment.cpp:61-157,288-320) on
//                        the compact sample in shared memory; k_tdist_cluster does
//                        K2a+K2b for <= 8 pairs over an 8-CTA cluster (latency mode).
//   K3  k_normal_eq_mma  jets (src/alignment.cpp:212-244), robust weights and the
//                        21+6+1 fp64 sums (src/alignment.cpp:321-335) on the FP64
//                        tensor cores (k_normal_eq: the FMA version).
//   K4  k_solve          fixed-order reduce, rank test, LDLT, SE(3) update, convergence
//                        (src/alignment.cpp:387-401) — no host round trip.
// Once per align: k_pyramid_slots, k_prep_A (A-side validity + gradients); the
// covariance pass adds k_bilateral_slots and k_covariance.
// Compiled with --fmad=false: mask-deciding arithmetic rounds exactly like the
// reference; reductions use a fixed tree (bit-reproducible run to run).
#include <cooperative_groups.h>
#include <cuda_runtime.h>
#include <math_constants.h>

#include <cmath>
#include <algorithm>
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

// ---------------------------------------------------------------------------
// Active-slot lists.  A converged slot (done_level == level) or a failed one
// skips the rest of the level, but its CTAs in the remaining launches of the
// graph would still be scheduled and exit: ~77 ns per CTA per SM whatever they do
// (tools/micro/empty_ctas.cu), i.e. 0.77 ms for the 1.47M CTAs of a 1024-slot
// level-0 K1 even when only 17 slots are left (bench level-0 iteration 10).
// k_active_slots compacts the slots still iterating, in slot order, before each
// K1, and picks the body of the iteration's K1 and K3 graph switch nodes: the
// same kernel over ceil(nslots / 2^k) slot rows, the smallest that covers the
// list (row j works on list entry j; rows past the count exit).  Body 0 is the
// plain one-row-per-slot grid (no list loads ahead of the slot check).
// slot of grid row j: list entry j (-1 past the count) or, without a list, j itself
template <bool LIST>
__device__ __forceinline__ int active_slot(const int* act, int j) {
  return LIST ? (j < act[0] ? act[1 + j] : -1) : j;
}

__global__ void __launch_bounds__(1024) k_active_slots(const SlotState* __restrict__ st, int nslots,
                                                       int level, int phase, int* __restrict__ act,
                                                       cudaGraphConditionalHandle h0,
                                                       cudaGraphConditionalHandle h1, int nbodies) {
  __shared__ int wsum[32];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  int base = 0;
  for (int s0 = 0; s0 < nslots; s0 += 1024) {
    const int s = s0 + (int)threadIdx.x;
    const bool on = s < nslots && slot_active(st[s], level, phase);
    const unsigned b = __ballot_sync(0xffffffffu, on);
    if (lane == 0) wsum[wid] = __popc(b);
    __syncthreads();
    int before = 0, total = 0;
    for (int k = 0; k < 32; ++k) {
      before += k < wid ? wsum[k] : 0;
      total += wsum[k];
    }
    if (on) act[1 + base + before + __popc(b & ((1u << lane) - 1u))] = s;
    base += total;
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    act[0] = base;
    if (nbodies > 0) {  // body k: ceil(nslots / 2^k) rows; none for an empty list
      int k = 0;
      while (k + 1 < nbodies && ((nslots + (2 << k) - 1) >> (k + 1)) >= base) ++k;
      const unsigned v = base == 0 ? (unsigned)nbodies : (unsigned)k;
      cudaGraphSetConditional(h0, v);
      cudaGraphSetConditional(h1, v);
    }
  }
}

void launch_active_slots(const AlignLaunch& a, int level, int phase, cudaStream_t s,
                         const SlotSwitch* sw) {
  if (!a.act) return;
  KScope ks_("active_slots", s);
  k_active_slots<<<1, 1024, 0, s>>>(a.st, a.nslots, level, phase, a.act, sw ? sw->h[0] : 0,
                                    sw ? sw->h[1] : 0, sw ? sw->nbodies : 0);
}


// Correctly rounded a / b from r = RN(1/b) (Markstein): q = RN(a r),
// e = a - b q (exact with FMA), RN(q + e r) == RN(a / b) for normal operands.
// Used where several quotients share a divisor; bit-identity with IEEE division
// is asserted by the warp-map tests and rgbid_selftest_division.
__device__ __forceinline__ double div_rcp(double a, double b, double r) {
  const double q = a * r;
  const double e = fma(-b, q, a);
  return fma(e, r, q);
}

// a / b correctly rounded: one IEEE reciprocal + the Markstein correction where the
// operands are in the range rgbid_selftest_division checks bit for bit, else a / b
__device__ __forceinline__ double div_safe(double a, double b) {
  const double mb = fabs(b), ma = fabs(a);
  if (mb > 1e-290 && mb < 1e290 && ma < 1e290 && (ma > 1e-280 || a == 0.0))
    return div_rcp(a, b, __drcp_rn(b));
  return a / b;
}

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

// bilinear fix-up for the warp's shared-tap evaluation of I_B and W_B.
// Fast path: the interpolation formula is evaluated directly; it is finite only
// if all four taps are finite (NaN/inf taps propagate through the products and
// sums, including 0 * inf), so the explicit tap checks of inc/image.hpp:59 are
// only needed when the result is non-finite — then the reference's hole (NaN)
// is returned if any tap is invalid, else the (overflowed) formula value.
__device__ __forceinline__ double bilin_fix(double r, double a, double b, double c, double d) {
  if (isfinite(r)) return r;
  return (valid(a) && valid(b) && valid(c) && valid(d)) ? r : CUDART_NAN;
}

// warp_px_iw on separate I_B, W_B maps (k_warp_maps: the C-ABI inverse_geometric_warp,
// whose frame B may differ in size from A).
__device__ __forceinline__ void warp_px(const WarpMats& m, const double* __restrict__ IB,
                                        const double* __restrict__ WB, int wb, int hb, int x,
                                        int y, double w_a, double& oI, double& oW, double& mx,
                                        double& my) {
  const bool v0 = valid(w_a) && w_a > 0.0;
  const double wa = v0 ? w_a : 1.0;
  const double qz = __drcp_rn(wa);  // == 1.0 / w_a
  const double qx = div_rcp((double)x, wa, qz), qy = div_rcp((double)y, wa, qz);
  const double xb0 = red3(m.Rt_BA[0] * qx, m.Rt_BA[1] * qy, m.Rt_BA[2] * qz) + m.tt_BA[0];
  const double xb1 = red3(m.Rt_BA[3] * qx, m.Rt_BA[4] * qy, m.Rt_BA[5] * qz) + m.tt_BA[1];
  const double xb2 = red3(m.Rt_BA[6] * qx, m.Rt_BA[7] * qy, m.Rt_BA[8] * qz) + m.tt_BA[2];
  const bool v1 = v0 && xb2 > 1e-12;
  const double z = v1 ? xb2 : 1.0;
  const double rz2 = __drcp_rn(z);
  const double px = div_rcp(xb0, z, rz2), py = div_rcp(xb1, z, rz2);
  mx = v1 ? px : CUDART_NAN;
  my = v1 ? py : CUDART_NAN;
  const bool inb = v1 && (px >= 0.0 && px <= wb - 1.0 && py >= 0.0 && py <= hb - 1.0);
  const double sx = inb ? px : 0.0, sy = inb ? py : 0.0;
  const int x0 = (int)floor(sx), y0 = (int)floor(sy);
  const int dx = x0 + 1 < wb ? 1 : 0;  // x1 = min(x0 + 1, w - 1)
  const int dy = y0 + 1 < hb ? wb : 0; // y1 = min(y0 + 1, h - 1)
  const double fx = sx - x0, fy = sy - y0, gx = 1 - fx, gy = 1 - fy;
  const int i00 = y0 * wb + x0;
  const double a00 = __ldg(IB + i00), a10 = __ldg(IB + i00 + dx), a01 = __ldg(IB + i00 + dy),
               a11 = __ldg(IB + i00 + dy + dx);
  const double b00 = __ldg(WB + i00), b10 = __ldg(WB + i00 + dx), b01 = __ldg(WB + i00 + dy),
               b11 = __ldg(WB + i00 + dy + dx);
  const double ri = bilin_fix(gy * (gx * a00 + fx * a10) + fy * (gx * a01 + fx * a11), a00, a10, a01, a11);
  const double w_meas = bilin_fix(gy * (gx * b00 + fx * b10) + fy * (gx * b01 + fx * b11), b00, b10, b01, b11);
  oI = inb ? ri : CUDART_NAN;
  const bool v2 = inb && valid(w_meas) && w_meas > 0.0;
  const double rz = red3(m.Rt_AB[6] * px, m.Rt_AB[7] * py, m.Rt_AB[8] * 1.0);
  const double za = div_safe(rz, v2 ? w_meas : 1.0) + m.tt_AB[2];
  const bool v3 = v2 && za > 1e-12;
  oW = v3 ? __drcp_rn(za) : CUDART_NAN;  // == 1.0 / za
}

// one A pixel of inverse_geometric_warp — src/warping.cpp:96-111 (bit-identical),
// on frame B stored interleaved {I, W}: the four bilinear taps are four 16-byte
// loads instead of eight 8-byte loads (-11% per level-0 launch).  Written branch-free (predicates + clamped, always-issued tap loads) so that
// several pixels unrolled in one thread overlap their gathers.
__device__ __forceinline__ void warp_px_iw(const WarpMats& m, const double2* __restrict__ IWB,
                                           int wb, int hb, double bx1, double by1, int x,
                                        int y, double w_a, double& oI, double& oW, double& mx,
                                        double& my) {
  const bool v0 = valid(w_a) && w_a > 0.0;
  const double wa = v0 ? w_a : 1.0;
  const double qz = __drcp_rn(wa);  // == 1.0 / w_a
  const double qx = div_rcp((double)x, wa, qz), qy = div_rcp((double)y, wa, qz);
  const double xb0 = red3(m.Rt_BA[0] * qx, m.Rt_BA[1] * qy, m.Rt_BA[2] * qz) + m.tt_BA[0];
  const double xb1 = red3(m.Rt_BA[3] * qx, m.Rt_BA[4] * qy, m.Rt_BA[5] * qz) + m.tt_BA[1];
  const double xb2 = red3(m.Rt_BA[6] * qx, m.Rt_BA[7] * qy, m.Rt_BA[8] * qz) + m.tt_BA[2];
  const bool v1 = v0 && xb2 > 1e-12;
  const double z = v1 ? xb2 : 1.0;
  const double rz2 = __drcp_rn(z);
  const double px = div_rcp(xb0, z, rz2), py = div_rcp(xb1, z, rz2);
  mx = v1 ? px : CUDART_NAN;
  my = v1 ? py : CUDART_NAN;
  // the bounds test as one predicate expression (no short-circuit branch) against
  // w - 1 and h - 1 as kernel-parameter doubles (constant-bank operands)
  const bool inb = v1 & (px >= 0.0) & (px <= bx1) & (py >= 0.0) & (py <= by1);
  const double sx = inb ? px : 0.0, sy = inb ? py : 0.0;
  const int x0 = (int)floor(sx), y0 = (int)floor(sy);
  const int dx = x0 + 1 < wb ? 1 : 0;  // x1 = min(x0 + 1, w - 1)
  const int dy = y0 + 1 < hb ? wb : 0; // y1 = min(y0 + 1, h - 1)
  const double fx = sx - x0, fy = sy - y0, gx = 1 - fx, gy = 1 - fy;
  const int i00 = y0 * wb + x0;
  const double2 t00 = __ldg(IWB + i00), t10 = __ldg(IWB + i00 + dx), t01 = __ldg(IWB + i00 + dy),
                t11 = __ldg(IWB + i00 + dy + dx);
  const double a00 = t00.x, a10 = t10.x, a01 = t01.x, a11 = t11.x;
  const double b00 = t00.y, b10 = t10.y, b01 = t01.y, b11 = t11.y;
  // the formula alone: it is non-finite exactly when the reference's result is a
  // hole (an invalid tap) or has overflowed, and K1's consumers (the validity tests,
  // the NaN-skipping downsample, K2's sample of valid residuals, K3's zeroed rows)
  // treat both alike -- only the payload of an invalid value differs (bilin_fix
  // keeps the reference's for the C-ABI warp maps)
  const double ri = gy * (gx * a00 + fx * a10) + fy * (gx * a01 + fx * a11);
  const double w_meas = gy * (gx * b00 + fx * b10) + fy * (gx * b01 + fx * b11);
  oI = inb ? ri : CUDART_NAN;
  const bool v2 = inb && valid(w_meas) && w_meas > 0.0;
  const double rz = red3(m.Rt_AB[6] * px, m.Rt_AB[7] * py, m.Rt_AB[8] * 1.0);
  const double za = rz / (v2 ? w_meas : 1.0) + m.tt_AB[2];  // IEEE division (the library's
                                                             // sequence beats div_safe here)
  const bool v3 = v2 && za > 1e-12;
  oW = v3 ? __drcp_rn(za) : CUDART_NAN;  // == 1.0 / za
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

// 2x2 NaN-aware mean — inc/image.hpp:73-91 (tap order (0,0),(1,0),(0,1),(1,1)).
// sum / n for n = 1, 2, 4 is the exact product sum * (1/n) (a power of two: the same
// correctly rounded value), so only n = 3 (a hole next to the block) divides.
__device__ __forceinline__ double ds4(double a, double b, double c, double d) {
  double sum = 0.0;
  int n = 0;
  if (valid(a)) sum += a, ++n;
  if (valid(b)) sum += b, ++n;
  if (valid(c)) sum += c, ++n;
  if (valid(d)) sum += d, ++n;
  if (n == 3) return sum / 3.0;
  return n == 4 ? sum * 0.25 : n == 2 ? sum * 0.5 : n == 1 ? sum : CUDART_NAN;
}

// ---------------------------------------------------------------------------
// K1: warp + downsample-to-level + jet validity + per-tile validity bitmasks.
// The A-side conditions of src/alignment.cpp:209-211,227 (valid/positive w_a,
// valid i_a, gradient_at(I_A), gradient_at(W_A)) do not change across IRLS
// iterations: they are precomputed once per alignment into amask (k_amask); K1
// adds the warped-B conditions and ballots the row-major validity bits per
// tile (compacted rank = prefix popcount, consumed by the sample gather of K2).
// thread layout of K1 at level L: k1_cw columns x k1_ng row groups (<= 256
// threads) over the tile's level-1 block (tx * 2^(L-1) columns x 2^(L-1) rows,
// <= 512 values); each thread computes 2^(L-1) / k1_ng level-1 values of four
// full-res warps each (512-thread CTAs at level 3 measured slower)
template <int L>
__host__ __device__ constexpr int k1_cw() {
  return (k1_tx(L) << (L - 1)) < 128 ? (k1_tx(L) << (L - 1)) : 128;
}
template <int L>
__host__ __device__ constexpr int k1_ng() {
  return (1 << (L - 1)) < 256 / k1_cw<L>() ? (1 << (L - 1)) : 256 / k1_cw<L>();
}
template <int L>
__host__ __device__ constexpr int k1_threads() { return k1_cw<L>() * k1_ng<L>(); }

// downsample2 applied K times to the 2^K x 2^K block of level-1 values at (r, c) of
// the staged tile (pitch cw), taps (0,0),(1,0),(0,1),(1,1) at every stage
template <int K>
__device__ __forceinline__ double ds_tree(const double* t, int cw, int r, int c) {
  if constexpr (K == 0) {
    return t[r * cw + c];
  } else {
    constexpr int hk = 1 << (K - 1);
    return ds4(ds_tree<K - 1>(t, cw, r, c), ds_tree<K - 1>(t, cw, r, c + hk),
               ds_tree<K - 1>(t, cw, r + hk, c), ds_tree<K - 1>(t, cw, r + hk, c + hk));
  }
}

template <int L, bool LIST>
#ifndef RGBID_K1_THREADS_PER_SM
#define RGBID_K1_THREADS_PER_SM 2048  // 32 registers, a full SM of threads: -4..7% per launch vs
                                      // 1536 (40 registers) since the warp lost its tap fix-up;
                                      // 1024 (64 registers) +8%
#endif
__global__ void __launch_bounds__(k1_threads<L>(), RGBID_K1_THREADS_PER_SM / k1_threads<L>()) k_warp_residuals(const SlotIO* __restrict__ io,
                                                           const SlotState* __restrict__ st,
                                                           LevelInfo li, int w0, int h0, int phase,
                                                           const int* __restrict__ act) {
  static_assert(L >= 1, "level 0 uses k_warp_residuals_l0");
  // grid (segment, level row, slot row): no tile-index division
  const int slot = active_slot<LIST>(act, blockIdx.z);
  if (slot < 0) return;
  const SlotState& S = st[slot];
  if (!slot_active(S, L, phase)) return;
  __shared__ WarpMats wm;
  if (threadIdx.x < 24)
    reinterpret_cast<double*>(&wm)[threadIdx.x] = reinterpret_cast<const double*>(&S.wm)[threadIdx.x];
  const SlotIO& o = io[slot];
  const double* __restrict__ WAw = phase ? o.fWA : o.WA[0];
  const double* __restrict__ IAl = phase ? o.fIA : o.IA[L];
  const uint8_t* __restrict__ am = o.amask[L];

  const int tid = threadIdx.x;
  const int seg = blockIdx.x, yl = blockIdx.y;
  const int tile = yl * li.nseg + seg;
  const int xl0 = seg * li.tx;
  const int nx = min(li.tx, li.w - xl0);
  // Level-1 block of the tile: cw = nx * 2^(L-1) columns (<= 128, one per thread) x
  // 2^(L-1) rows.  Each level-1 pixel = downsample2 of its 2x2 full-res warps,
  // computed in registers (4 independent gather chains), taps in the reference
  // order (0,0),(1,0),(0,1),(1,1) (inc/image.hpp:77-85).
  __shared__ double sI[512], sW[512];
  constexpr int CW = k1_cw<L>(), NG = k1_ng<L>();  // thread columns x row groups
  const int cw = nx << (L - 1);
  const int col = tid % CW, grp = tid / CW;
  const int x = (xl0 << L) + 2 * col;
  // one quad per thread (levels 1-2): its W_A values in flight while the warp
  // matrices arrive (at level 3 the extra registers cost more than they save)
  constexpr bool kHoist = (1 << (L - 1)) / NG == 1;
  double wa0[4];
#pragma unroll
  for (int q = 0; q < 4; ++q)
    wa0[q] = kHoist && col < cw ? __ldg(WAw + ((yl << L) + 2 * grp + (q >> 1)) * w0 + x + (q & 1))
                                : 0.0;
  __syncthreads();
  if (col < cw) {
#pragma unroll
    for (int rr = 0; rr < (1 << (L - 1)) / NG; ++rr) {
      const int r = rr * NG + grp;
      const int y = (yl << L) + 2 * r;
      double vi[4], vw[4], d0, d1;
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int xx = x + (q & 1), yy = y + (q >> 1);
        const double w_a = kHoist ? wa0[q] : __ldg(WAw + yy * w0 + xx);
        warp_px_iw(wm, o.IWB, w0, h0, li.bx1, li.by1, xx, yy, w_a, vi[q], vw[q], d0, d1);
      }
      sI[r * cw + col] = ds4(vi[0], vi[1], vi[2], vi[3]);
      sW[r * cw + col] = ds4(vw[0], vw[1], vw[2], vw[3]);
    }
  }
  __syncthreads();
  // remaining downsample stages (level 1 -> L) by the level-L pixel's own thread, in
  // registers from the staged level-1 values, in the reference's tap order at every
  // stage: no further block barrier
  double vI = 0.0, vW = 0.0;
  if (tid < nx) {
    vI = ds_tree<L - 1>(sI, cw, 0, tid << (L - 1));
    vW = ds_tree<L - 1>(sW, cw, 0, tid << (L - 1));
  }

  bool jet = false, dep = false;
  if (tid < nx) {
    const int idx = yl * li.w + xl0 + tid;
    const double ib = vI, wb = vW;
    o.ibw[idx] = make_double2(ib - __ldg(IAl + idx), wb);  // r_I (src/alignment.cpp:222), w_b
    const unsigned a = __ldg(am + idx);
    jet = (a & 1u) && valid(ib);
    dep = jet && (a & 2u) && valid(wb) && wb > 0.0;
  }
  const unsigned bj = __ballot_sync(0xffffffffu, jet), bd = __ballot_sync(0xffffffffu, dep);
  __shared__ int wcnt[2][4];
  const int lane = tid & 31, wid = tid >> 5;
  if (lane == 0 && wid < 4) {  // level pixels live in the first 128 threads
    wcnt[0][wid] = __popc(bj);
    wcnt[1][wid] = __popc(bd);
    o.bitsI[tile * kWordsPerTile + wid] = bj;
    o.bitsW[tile * kWordsPerTile + wid] = bd;
  }
  __syncthreads();
  if (tid == 0) {
    o.cntI[tile] = wcnt[0][0] + wcnt[0][1] + wcnt[0][2] + wcnt[0][3];
    o.cntW[tile] = wcnt[1][0] + wcnt[1][1] + wcnt[1][2] + wcnt[1][3];
  }
}

// Level-0 K1: 128 threads per 256-pixel tile, two independent pixels per thread
// (x and x + 128) so their dependent load chains (W_A -> gathers) overlap; a CTA
// takes the same segment of RGBID_K1L0_ROWS consecutive rows (one tile per 128
// threads), so the per-CTA setup -- slot check, warp matrices, barriers -- is shared.
#ifndef RGBID_K1L0_MINB
#define RGBID_K1L0_MINB 12
#endif
#ifndef RGBID_K1L0_ROWS
#define RGBID_K1L0_ROWS 1  // 2 and 4 rows per CTA measured 2.5% / 14% slower per launch
#endif
constexpr int kK1L0Rows = RGBID_K1L0_ROWS;
template <bool LIST>
__global__ void __launch_bounds__(128 * kK1L0Rows, RGBID_K1L0_MINB / kK1L0Rows)
    k_warp_residuals_l0(const SlotIO* __restrict__ io, const SlotState* __restrict__ st,
                        LevelInfo li, int w0, int h0, int phase, const int* __restrict__ act) {
  // grid (segment, row group, slot row): no tile-index division
  const int slot = active_slot<LIST>(act, blockIdx.z);
  if (slot < 0) return;
  const SlotState& S = st[slot];
  if (!slot_active(S, 0, phase)) return;
  __shared__ WarpMats wm;
  if (threadIdx.x < 24)
    reinterpret_cast<double*>(&wm)[threadIdx.x] = reinterpret_cast<const double*>(&S.wm)[threadIdx.x];
  const SlotIO& o = io[slot];
  const double* __restrict__ WAw = phase ? o.fWA : o.WA[0];
  const double* __restrict__ IA0 = phase ? o.fIA : o.IA[0];
  const uint8_t* __restrict__ am = o.amask[0];
  const int half = threadIdx.x >> 7, tid = threadIdx.x & 127;
  const int seg = blockIdx.x, yl = blockIdx.y * kK1L0Rows + half;
  const int tile = yl * li.nseg + seg;
  const int xl0 = seg * li.tx;
  const int nx = yl < li.h ? min(li.tx, li.w - xl0) : 0;
  // the pixels' A-side values in flight while the warp matrices arrive
  double wa[2], iav[2];
  unsigned amv[2];
#pragma unroll
  for (int q = 0; q < 2; ++q) {
    const int lx = tid + 128 * q;
    const int idx = yl * w0 + xl0 + lx;
    const bool in = lx < nx;
    wa[q] = in ? __ldg(WAw + idx) : 0.0;
    iav[q] = in ? __ldg(IA0 + idx) : 0.0;
    amv[q] = in ? __ldg(am + idx) : 0u;
  }
  __syncthreads();
  bool jet[2], dep[2];
#pragma unroll
  for (int q = 0; q < 2; ++q) {
    const int lx = tid + 128 * q;
    jet[q] = dep[q] = false;
    if (lx < nx) {
      const int idx = yl * w0 + xl0 + lx;
      const unsigned a = amv[q];
      const double ia = iav[q];
      double ib, wb, d0, d1;
      warp_px_iw(wm, o.IWB, w0, h0, li.bx1, li.by1, xl0 + lx, yl, wa[q], ib, wb, d0, d1);
      o.ibw[idx] = make_double2(ib - ia, wb);  // r_I (src/alignment.cpp:222), w_b: K2, K3
      jet[q] = (a & 1u) && valid(ib);
      dep[q] = jet[q] && (a & 2u) && valid(wb) && wb > 0.0;
    }
  }
  __shared__ int wcnt[kK1L0Rows][2][8];
  const int lane = tid & 31, wid = tid >> 5;
#pragma unroll
  for (int q = 0; q < 2; ++q) {
    const unsigned bj = __ballot_sync(0xffffffffu, jet[q]), bd = __ballot_sync(0xffffffffu, dep[q]);
    if (lane == 0 && yl < li.h) {
      const int word = wid + 4 * q;  // pixels [32 word, 32 word + 32) of the tile
      wcnt[half][0][word] = __popc(bj);
      wcnt[half][1][word] = __popc(bd);
      o.bitsI[tile * kWordsPerTile + word] = bj;
      o.bitsW[tile * kWordsPerTile + word] = bd;
    }
  }
  __syncthreads();
  if (tid == 0 && yl < li.h) {
    int tI = 0, tW = 0;
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      tI += wcnt[half][0][k];
      tW += wcnt[half][1][k];
    }
    o.cntI[tile] = tI;
    o.cntW[tile] = tW;
  }
}

// A-side part of residuals_and_jacobians, constant over the IRLS iterations:
// validity (src/alignment.cpp:209-211,227) and gradient_at of I_A and W_A
// (src/alignment.cpp:165-191) per level pixel.  phase 1 = from the filtered A
// into the level-0 slots (covariance pass, after the level loop).
// Tiled: a 32 x 8 pixel tile per CTA with its 1-pixel halo of I_A and W_A staged
// in shared memory (coalesced row loads, NaN outside the image = the reference's
// out-of-bounds hole), so every 3 x 3 stencil read is a shared load.
#ifndef RGBID_PREP_ROWS
#define RGBID_PREP_ROWS 4  // tile rows per thread (32 x 8 threads)
#endif
constexpr int kPTT = 8;                                   // thread rows
constexpr int kPTW = 32, kPTH = kPTT * RGBID_PREP_ROWS, kPRW = kPTW + 2, kPRH = kPTH + 2;

// gradient_at on the staged tile (same tests and expressions)
__device__ __forceinline__ bool grad_sm(const double* t, int i, double& gx, double& gy) {
  const double c = t[i];
  if (!valid(c)) return false;
  const double l = t[i - 1], r = t[i + 1];
  if (valid(l) && valid(r))
    gx = (r - l) / 2.0;
  else if (valid(r))
    gx = r - c;
  else if (valid(l))
    gx = c - l;
  else
    return false;
  const double u = t[i - kPRW], d = t[i + kPRW];
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

__global__ void __launch_bounds__(kPTW * kPTT) k_prep_A(const SlotIO* __restrict__ io,
                                                         const SlotState* __restrict__ st,
                                                         int level, int w, int h, int phase) {
  const int slot = blockIdx.z;
  if (st[slot].status != RGBID_OK) return;
  const SlotIO& o = io[slot];
  const double* IA = phase ? o.fIA : o.IA[level];
  const double* WA = phase ? o.fWA : o.WA[level];
  __shared__ double tI[kPRW * kPRH], tW[kPRW * kPRH];
  const int x0 = blockIdx.x * kPTW, y0 = blockIdx.y * kPTH, t = threadIdx.x;
  constexpr int NT = kPTW * kPTT;
  constexpr int kLoads = (kPRW * kPRH + NT - 1) / NT;
#pragma unroll
  for (int j = 0; j < kLoads; ++j) {  // the halo'd tile, all loads of a thread in flight
    const int i = t + j * NT;
    if (i < kPRW * kPRH) {
      const int ry = i / kPRW, rx = i - ry * kPRW;
      const int gx = x0 - 1 + rx, gy = y0 - 1 + ry;
      const bool in = gx >= 0 && gx < w && gy >= 0 && gy < h;
      const size_t k = (size_t)gy * w + gx;
      tI[i] = in ? __ldg(IA + k) : CUDART_NAN;
      tW[i] = in ? __ldg(WA + k) : CUDART_NAN;
    }
  }
  __syncthreads();
  const int tx = t % kPTW, x = x0 + tx;
#pragma unroll
  for (int rr = 0; rr < RGBID_PREP_ROWS; ++rr) {
    const int ty = t / kPTW + rr * kPTT, y = y0 + ty;
    if (x >= w || y >= h) continue;
    const int i = (ty + 1) * kPRW + tx + 1;
    const size_t k = (size_t)y * w + x;
    const double w_a = tW[i], i_a = tI[i];
    double g[4] = {0.0, 0.0, 0.0, 0.0};
    unsigned m = 0;
    if (valid(w_a) && w_a > 0.0 && valid(i_a) && grad_sm(tI, i, g[0], g[1])) m |= 1u;
    if (grad_sm(tW, i, g[2], g[3])) m |= 2u;
    o.amask[level][k] = (uint8_t)m;
    double2* gp = reinterpret_cast<double2*>(o.agrad[level] + 4 * k);
    gp[0] = make_double2(g[0], g[1]);
    gp[1] = make_double2(g[2], g[3]);
  }
}

// frame B interleaved {I, W} for K1's taps, once per align
__global__ void k_interleave_B(const SlotIO* __restrict__ io, const SlotState* __restrict__ st,
                               int n) {
  const int slot = blockIdx.y;
  if (st[slot].status != RGBID_OK) return;
  const SlotIO& o = io[slot];
  // two pixels per thread: 16-byte loads of I_B and W_B where the pair is aligned
  const int k = 2 * (blockIdx.x * blockDim.x + threadIdx.x);
  if (k + 1 < n && ((reinterpret_cast<size_t>(o.IB) | reinterpret_cast<size_t>(o.WB)) & 15) == 0) {
    const double2 i2 = __ldg(reinterpret_cast<const double2*>(o.IB + k));
    const double2 w2 = __ldg(reinterpret_cast<const double2*>(o.WB + k));
    o.IWB[k] = make_double2(i2.x, w2.x);
    o.IWB[k + 1] = make_double2(i2.y, w2.y);
  } else {
    for (int j = k; j < min(k + 2, n); ++j) o.IWB[j] = make_double2(__ldg(o.IB + j), __ldg(o.WB + j));
  }
}

void launch_interleave_B(const AlignLaunch& a, cudaStream_t s) {
  KScope ks_("interleave_B", s);
  const int n = a.w0 * a.h0;
  k_interleave_B<<<dim3((n + 511) / 512, a.nslots), 256, 0, s>>>(a.io, a.st, n);
}

void launch_amask(const AlignLaunch& a, int levels, int phase, cudaStream_t s) {
  for (int l = 0; l < levels; ++l) {
    const int w = a.w0 >> l, h = a.h0 >> l;
    KScope ks_("prep_A", s);
    k_prep_A<<<dim3((w + kPTW - 1) / kPTW, (h + kPTH - 1) / kPTH, a.nslots), kPTW * kPTT, 0, s>>>(
        a.io, a.st, l, w, h, phase);
  }
}

// pyramid levels 1..L-1 of every slot whose frame A needs them (src/alignment.cpp:13-28)
__global__ void k_pyramid_slots(const SlotIO* __restrict__ io, int level, int w, int h) {
  const SlotIO& o = io[blockIdx.y];
  if (!o.build_pyr) return;
  const int ow = w / 2, oh = h / 2;
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= ow * oh) return;
  const int y = k / ow, x = k - y * ow;
  const double* I = o.IA[level - 1];
  const double* W = o.WA[level - 1];
  const int i0 = (2 * y) * w + 2 * x, i1 = i0 + w;
  o.IA[level][k] = ds4(I[i0], I[i0 + 1], I[i1], I[i1 + 1]);
  o.WA[level][k] = ds4(W[i0], W[i0 + 1], W[i1], W[i1 + 1]);
}

void launch_pyramid_slots(const AlignLaunch& a, int levels, cudaStream_t s) {
  for (int l = 1; l < levels; ++l) {
    const int w = a.w0 >> (l - 1), h = a.h0 >> (l - 1);
    const int n = (w / 2) * (h / 2);
    KScope ks_("pyramid", s);
    k_pyramid_slots<<<dim3((n + 255) / 256, a.nslots), 256, 0, s>>>(a.io, l, w, h);
  }
}

static const char* kLevelNames[2][kMaxLevels] = {
    {"warp_residuals_L0", "warp_residuals_L1", "warp_residuals_L2", "warp_residuals_L3",
     "warp_residuals_L4", "warp_residuals_L5"},
    {"warp_residuals_cov", "warp_residuals_cov", "warp_residuals_cov", "warp_residuals_cov",
     "warp_residuals_cov", "warp_residuals_cov"}};

void launch_warp_residuals(const AlignLaunch& a, const LevelInfo& li, int phase, cudaStream_t s,
                           int rows) {
  KScope ks_(kLevelNames[phase ? 1 : 0][li.level], s);
  const int rows0 = (li.h + kK1L0Rows - 1) / kK1L0Rows;
  dim3 grid(li.nseg, li.h, rows > 0 ? rows : a.nslots);  // tile = row * nseg + segment
  const int* act = a.act;
  const bool list = rows > 0 && act;  // rows = 0: one row per slot, no list
#define K1L(L)                                                                                  \
  (list ? k_warp_residuals<L, true><<<grid, k1_threads<L>(), 0, s>>>(a.io, a.st, li, a.w0, a.h0, \
                                                                     phase, act)               \
        : k_warp_residuals<L, false><<<grid, k1_threads<L>(), 0, s>>>(a.io, a.st, li, a.w0,     \
                                                                      a.h0, phase, act))
  switch (li.level) {
    case 0: {
      const dim3 g0(li.nseg, rows0, grid.z);
      if (list)
        k_warp_residuals_l0<true><<<g0, 128 * kK1L0Rows, 0, s>>>(a.io, a.st, li, a.w0, a.h0, phase, act);
      else
        k_warp_residuals_l0<false><<<g0, 128 * kK1L0Rows, 0, s>>>(a.io, a.st, li, a.w0, a.h0, phase, act);
      break;
    }
    case 1: K1L(1); break;
    case 2: K1L(2); break;
    case 3: K1L(3); break;
    case 4: K1L(4); break;
    case 5: K1L(5); break;
    default: return;
  }
#undef K1L
}

// ---------------------------------------------------------------------------
// K2: Student-t chain.  One CTA (kTdistThreads) per (slot, residual type).  The
// systematic sample (src/alignment.cpp:50-57) is gathered into shared memory
// (fixed per-thread ownership -> deterministic), then the whole
// chain of src/alignment.cpp:61-157,288-320 runs with block-wide fixed-order
// reductions.  Per-sample arithmetic uses (v - mu) * (1/sigma) and a
// MUFU-seeded Newton reciprocal for t_weight (<= 1-2 ulp per term; the
// reference's sums are sequential, ours a fixed tree — both only change
// rounding, well inside the 1e-4 normal-equation tolerance).

// Block-wide sum; every thread receives the bit-identical total.  The scratch
// has two halves used alternately (the caller's parity flips per call), so one
// barrier per reduction suffices: a half is rewritten only two calls later,
// after every thread has passed the intervening barrier.
template <int NV, int NT>
__device__ __forceinline__ void block_allsum(double (&v)[NV], double* scratch2, int& parity) {
  constexpr int NW = NT / 32;
  double* scratch = scratch2 + parity * (NW * 2);
  parity ^= 1;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
#pragma unroll
  for (int off = 16; off > 0; off >>= 1)
#pragma unroll
    for (int i = 0; i < NV; ++i) v[i] += __shfl_xor_sync(0xffffffffu, v[i], off);
  if (lane == 0)
#pragma unroll
    for (int i = 0; i < NV; ++i) scratch[wid * NV + i] = v[i];
  __syncthreads();
  // lane l takes warp l % NW's partial (what a 5-round butterfly over zero-padded lanes
  // holds after its rounds xor >= NW, which only add zeros), so log2(NW) rounds finish
  // the same sum (the same additions in the same order, up to the sign of an exact zero)
#pragma unroll
  for (int i = 0; i < NV; ++i) v[i] = scratch[(lane % NW) * NV + i];
#pragma unroll
  for (int off = NW / 2; off > 0; off >>= 1)
#pragma unroll
    for (int i = 0; i < NV; ++i) v[i] += __shfl_xor_sync(0xffffffffu, v[i], off);
}

struct TD {
  double mu, sigma, nu;
};

// Phase counters for the Student-t chain (thread 0 of each CTA; instrumented
// builds only: RGBID_NVFLAGS=-DRGBID_TDIST_TRACE, read by tools/tdist_phases.py)
#ifdef RGBID_TDIST_TRACE
__device__ unsigned long long g_tph[24];
#define TPH_T(v) const unsigned long long v = clock64()
#define TPH_ADD(i, t0) \
  if (threadIdx.x == 0) atomicAdd(&g_tph[i], (unsigned long long)(clock64() - (t0)))
#define TPH_CNT(i, n) \
  if (threadIdx.x == 0) atomicAdd(&g_tph[i], (unsigned long long)(n))
#else
#define TPH_T(v)
#define TPH_ADD(i, t0)
#define TPH_CNT(i, n)
#endif

struct Sample;
template <int NV, int NT>
__device__ __forceinline__ void sample_allsum(double (&v)[NV], Sample& S);

__device__ __forceinline__ double t_weight(double x, double nu) { return (nu + 1.0) / (nu + x * x); }

// 1/q for q >= 1 (t_weight denominators): MUFU seed + cubic Newton step (full precision).
__device__ __forceinline__ double rcp_fast(double q) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(q));
  const double e = fma(-q, r, 1.0);
  return fma(r, fma(e, e, e), r);
}
// 1/q for normal positive q: MUFU seed + one quadratic Newton step (~1e-12 relative;
// used only inside sums whose order already differs from the reference).
__device__ __forceinline__ double rcp_q(double q) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(q));
  return fma(r, fma(-q, r, 1.0), r);
}

struct Sample {
  const double* v;  // shared memory; thread t owns v[t], v[t + NT], ... (this CTA's share)
  double* scratch;  // 2 x (NT/32 x 2) doubles for block_allsum
  int parity;
  int m;            // sample size (all CTAs of the cluster)
  int m_local;      // samples held by this CTA
  int kfull;        // rounds where every thread owns a sample (m_local / NT)
  int cs;           // cluster size sharing the sample (1 = single CTA)
  double* cbuf;     // this CTA's [2][kTdistCluster * NW * 2] warp-partial slots (cluster mode)
  uint64_t* cmbar;  // this CTA's two mbarriers guarding cbuf's halves (cluster mode)
  int cred;         // cluster reductions done
  int rank;         // this CTA's rank in the cluster
  // memo of the last estimate_location_scale(nu) call: same sample + same nu
  // -> same result (e.g. the final refit repeating estimate_nu's, src/alignment.cpp:117,316)
  double memo_nu;
  TD memo;
  // the sample's mean and root-mean-square deviation (the start of every
  // estimate_location_scale call, src/alignment.cpp:65-71): computed once per chain
  bool have_mom;
  double mu0, sigma0;
};

// Cluster-wide sum (latency mode): every warp's lane d pushes the warp's partials
// into CTA d's slot array with st.async, completing transaction bytes on CTA d's
// mbarrier; each CTA waits on its own mbarrier, then reduces the CS x NW slots in
// a fixed tree -- identical bits in every thread of every CTA, with no block or
// cluster barrier.  The slots and mbarriers are double buffered: a CTA cannot run
// two reductions ahead of a peer (its reduction r+1 needs the peer's r+1
// partials, sent only after the peer consumed r).
template <int NV, int NT>
__device__ __forceinline__ void cluster_allsum(double (&v)[NV], Sample& S) {
  constexpr int NW = NT / 32, CS = kTdistCluster, NP = CS * NW;
  static_assert(NP % 32 == 0 && CS <= 32, "whole slots per lane in the final tree");
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int p = S.cred & 1;
  const unsigned ph = (unsigned)(S.cred >> 1) & 1u;
  ++S.cred;
#pragma unroll
  for (int off = 16; off > 0; off >>= 1)
#pragma unroll
    for (int i = 0; i < NV; ++i) v[i] += __shfl_xor_sync(0xffffffffu, v[i], off);
  double* buf = S.cbuf + p * (NP * 2);
  uint64_t* mb = S.cmbar + p;
  if (threadIdx.x == 0) {
    const unsigned a = (unsigned)__cvta_generic_to_shared(mb);
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(a),
                 "r"((unsigned)(NP * NV * 8))
                 : "memory");
  }
  if (lane < CS) {
    unsigned rem_buf, rem_mb;
    const unsigned lb = (unsigned)__cvta_generic_to_shared(buf + (S.rank * NW + wid) * NV);
    const unsigned lm = (unsigned)__cvta_generic_to_shared(mb);
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(rem_buf) : "r"(lb), "r"(lane));
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(rem_mb) : "r"(lm), "r"(lane));
#pragma unroll
    for (int i = 0; i < NV; ++i)
      asm volatile(
          "st.async.shared::cluster.mbarrier::complete_tx::bytes.b64 [%0], %1, [%2];" ::"r"(
              rem_buf + 8 * i),
          "l"(__double_as_longlong(v[i])), "r"(rem_mb)
          : "memory");
  }
  {
    const unsigned a = (unsigned)__cvta_generic_to_shared(mb);
    unsigned done = 0;
    do {
      asm volatile(
          "{ .reg .pred P; mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 P, [%1], %2;"
          " selp.u32 %0, 1, 0, P; }"
          : "=r"(done)
          : "r"(a), "r"(ph)
          : "memory");
    } while (!done);
  }
#pragma unroll
  for (int i = 0; i < NV; ++i) {
    double t = buf[lane * NV + i];
#pragma unroll
    for (int j = 1; j < NP / 32; ++j) t += buf[(lane + 32 * j) * NV + i];
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) t += __shfl_xor_sync(0xffffffffu, t, off);
    v[i] = t;
  }
}

// Sum over the whole sample: fixed-order block reduction (single CTA), or the
// cluster-wide push reduction (latency mode).  Every thread of every CTA ends
// with the bit-identical total.
template <int NV, int NT>
__device__ __forceinline__ void sample_allsum(double (&v)[NV], Sample& S) {
  TPH_T(tr0);
  if constexpr (NT == kTdistClusterThreads) {
    if (S.cs > 1)
      cluster_allsum<NV, NT>(v, S);
    else
      block_allsum<NV, NT>(v, S.scratch, S.parity);
  } else {
    block_allsum<NV, NT>(v, S.scratch, S.parity);
  }
  TPH_ADD(8, tr0);
  TPH_CNT(9, 1);
}

// sum over the thread's samples of f(v): bodies of 8 independent samples into
// 4 accumulators (the per-sample chains are latency-bound with one CTA per SM);
// fixed assignment -> deterministic
template <int NT, int NV, typename F>
__device__ __forceinline__ void sample_sum(const Sample& S, double (&acc)[NV], F f) {
  double a[4][NV];
#pragma unroll
  for (int j = 0; j < 4; ++j)
#pragma unroll
    for (int i = 0; i < NV; ++i) a[j][i] = 0.0;
  const double* v = S.v + threadIdx.x;
  int k = 0;
  for (; k + 7 < S.kfull; k += 8) {
    double x[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) x[u] = v[(k + u) * NT];
#pragma unroll
    for (int u = 0; u < 8; ++u) f(x[u], a[u & 3]);
  }
  for (; k * NT < S.m_local; ++k)
    if (k * NT + (int)threadIdx.x < S.m_local) f(v[k * NT], a[0]);
#pragma unroll
  for (int i = 0; i < NV; ++i) acc[i] = (a[0][i] + a[1][i]) + (a[2][i] + a[3][i]);
}

// Running product of positive normal doubles kept as mantissa in [1,2) and an
// integer binary exponent: sum(log q) = log(mantissa) + E ln2 with one log per
// thread.  Rounding: one ulp per multiply (k ulps over k factors), the same order
// as summing k correctly-rounded logs.  `bad` latches a non-normal intermediate.
struct LogProd {
  double p = 1.0;
  int e = 0;
  bool bad = false;
  __device__ __forceinline__ void renorm() {
    const long long b = __double_as_longlong(p);
    const int ex = (int)((unsigned long long)b >> 52);  // p > 0: sign bit clear
    bad |= (ex == 0) | (ex == 0x7ff);
    e += ex - 1023;
    p = __longlong_as_double((b & 0x000FFFFFFFFFFFFFll) | 0x3FF0000000000000ll);
  }
};

// Sums over the thread's samples of r = 1/q, q = (v-mu)^2 + c1 (> 0), and
// optionally of r v (WV) and log q (WL).  kQBody (4) samples form one fraction
// N/D (pairwise tree, D = prod q): one reciprocal per 4 samples instead of 4
// (the FP64 MUFU reciprocal issues at a quarter of the DFMA rate; 8 per fraction
// measured 1.5% slower in the batch kernel, 10% in latency mode), all terms
// positive except r v's numerators.  D also feeds the running log-product, so
// sum(log q) costs one log per thread.  A thread whose sums show an out-of-range
// fraction (a non-finite or zero sum of positive terms, or a non-normal log
// product: only for |v - mu| beyond ~1e38 or q below ~1e-77) redoes its share with
// exact per-sample division and logs.
#ifndef RGBID_QBODY
#define RGBID_QBODY 4
#endif
constexpr int kQBody = RGBID_QBODY;  // samples per fraction
#ifndef RGBID_QUNROLL
#define RGBID_QUNROLL 2
#endif
constexpr int kQUnroll = RGBID_QUNROLL;  // bodies per loop trip

// sum_i 1/q_i = N/D (and sum_i x_i/q_i = NV/D) over BW samples, pairwise tree
template <int BW, bool WV>
__device__ __forceinline__ void frac_tree(const double (&q)[BW], const double (&x)[BW], double& D,
                                          double& NR, double& NV) {
  double d[BW / 2], n[BW / 2], mv[BW / 2];
#pragma unroll
  for (int i = 0; i < BW / 2; ++i) {
    d[i] = q[2 * i] * q[2 * i + 1];
    n[i] = q[2 * i] + q[2 * i + 1];
    if (WV) mv[i] = fma(x[2 * i], q[2 * i + 1], x[2 * i + 1] * q[2 * i]);
  }
#pragma unroll
  for (int w = BW / 2; w > 1; w >>= 1)
#pragma unroll
    for (int i = 0; i < w / 2; ++i) {
      n[i] = fma(n[2 * i], d[2 * i + 1], n[2 * i + 1] * d[2 * i]);
      if (WV) mv[i] = fma(mv[2 * i], d[2 * i + 1], mv[2 * i + 1] * d[2 * i]);
      d[i] = d[2 * i] * d[2 * i + 1];
    }
  D = d[0];
  NR = n[0];
  if (WV) NV = mv[0];
}

// one body of q_sums: BW samples k..k+BW-1 of this thread; MASKED pads the
// samples past m_local with q = 1, x = 0 (1/q = 1 each, subtracted by the caller;
// log 1 = 0; x/q = 0)
template <int NT, int BW, bool WV, bool WL, bool MASKED>
__device__ __forceinline__ void q_body(const Sample& S, const double* v, int k, double mu, double c1,
                                       double& sr, double& sv, LogProd& P, bool& bad) {
  double x[BW], q[BW];
#pragma unroll
  for (int u = 0; u < BW; ++u) {
    const bool ok = !MASKED || (k + u) * NT + (int)threadIdx.x < S.m_local;
    x[u] = ok ? v[(k + u) * NT] : 0.0;
    const double d = x[u] - mu;
    q[u] = ok ? fma(d, d, c1) : 1.0;
  }
  double D, NR, NV;
  frac_tree<BW, WV>(q, x, D, NR, NV);
  const double inv = rcp_fast(D);
  sr = fma(NR, inv, sr);
  if (WV) sv = fma(NV, inv, sv);
  if (WL) {
    P.p *= D;
    P.renorm();
  }
}

template <int NT, bool WV, bool WL>
__device__ __forceinline__ void q_sums(const Sample& S, double mu, double c1, double (&out)[3]) {
  constexpr int BW = kQBody;
  const double* v = S.v + threadIdx.x;
  double sr = 0.0, sv = 0.0, slog = 0.0;
  LogProd P;
  bool bad = false;
  int k = 0;
#pragma unroll kQUnroll
  for (; k + BW - 1 < S.kfull; k += BW)  // branch-free bodies
    q_body<NT, BW, WV, WL, false>(S, v, k, mu, c1, sr, sv, P, bad);
  const int kend = (S.m_local + NT - 1) / NT;
  for (; k < kend; k += BW) {  // the rest, padded
    q_body<NT, BW, WV, WL, true>(S, v, k, mu, c1, sr, sv, P, bad);
    int npad = 0;
#pragma unroll
    for (int u = 0; u < BW; ++u) npad += (k + u) * NT + (int)threadIdx.x < S.m_local ? 0 : 1;
    sr -= (double)npad;
  }
  // out-of-range fractions show in the thread's sums: an overflowing or vanishing D
  // (|v - mu| beyond ~1e38 or q below ~1e-77) leaves a non-finite or zero sum of
  // strictly positive terms; anything less extreme stays within rounding
  bad |= !(sr > 0.0 && sr < 1.0e300) || (WV && !isfinite(sv));
  if (bad) {  // exact per-sample division for this thread's share
    sr = sv = 0.0;
    for (int kk = 0; kk * NT < S.m_local; ++kk)
      if (kk * NT + (int)threadIdx.x < S.m_local) {
        const double x = v[kk * NT], d = x - mu, q = fma(d, d, c1), r = 1.0 / q;
        sr += r;
        if (WV) sv = fma(r, x, sv);
        if (WL) slog += log(q);
      }
  }
  out[0] = sr;
  out[1] = sv;
  if (WL) {
    if (bad) {
      out[2] = slog;
    } else {
      const double E = (double)P.e;  // E * ln2_hi exact (ln2_hi has 21 trailing zero bits)
      out[2] = log(P.p) + (E * 6.93147180369123816490e-01 + E * 1.90821492927058770002e-10);
    }
  }
}

// estimate_location_scale on the shared-memory sample — src/alignment.cpp:61-101
template <int NT>
__device__ __forceinline__ TD loc_scale(Sample& S, double nu, double* scratch) {
  TD p{0.0, 1.0, nu};
  const int m = S.m;
  if (m == 0) return p;
  if (S.memo_nu == nu) return S.memo;
  TPH_T(tl0);
  TPH_CNT(2, 1);
  const double inv_m = 1.0 / (double)m;
  double a1[1];
  if (!S.have_mom) {
    sample_sum<NT>(S, a1, [](double v, double (&a)[1]) { a[0] += v; });
    sample_allsum<1, NT>(a1, S);
    const double mu0 = a1[0] / (double)m;
    sample_sum<NT>(S, a1, [mu0](double v, double (&a)[1]) {
      const double d = v - mu0;
      a[0] = fma(d, d, a[0]);
    });
    sample_allsum<1, NT>(a1, S);
    S.mu0 = mu0;
    S.sigma0 = sqrt(a1[0] / (double)m);
    S.have_mom = true;
  }
  double mu = S.mu0;
  double sigma = S.sigma0;
  TD out;
  if (sigma < 1e-8) {
    out = TD{mu, 1e-8, nu};
  } else {
    const double nu1 = nu + 1.0;
    for (int it = 0; it < 50; ++it) {
      // t_weight((v-mu)/sigma, nu) = c2 / (c1 + (v-mu)^2), c1 = nu s2, c2 = (nu+1) s2;
      // the constant c2 is applied after the reduction (sums of r = 1/(c1 + d^2))
      const double s2 = sigma * sigma, c1 = nu * s2, c2 = nu1 * s2;
      double a3[3];
      q_sums<NT, true, false>(S, mu, c1, a3);
      double a2[2] = {a3[0], a3[1]};
      sample_allsum<2, NT>(a2, S);
      const double mu_new = a2[1] / a2[0];  // (c2 sum r v) / (c2 sum r)
      // sum w d^2 = c2 sum d^2 / (d^2 + c1) = c2 (m - c1 sum r)
      q_sums<NT, false, false>(S, mu_new, c1, a3);
      a1[0] = a3[0];
      sample_allsum<1, NT>(a1, S);
      a1[0] = c2 * fma(-c1, a1[0], (double)m);
      const double sigma_new = dmax_std(1e-8, sqrt(a1[0] * inv_m));
      const double rel = fabs(sigma_new - sigma) / sigma;
      mu = mu_new;
      sigma = sigma_new;
      TPH_CNT(3, 1);
      if (rel < 1e-4) break;
    }
    out = TD{mu, dmax_std(sigma, 1e-8), nu};
  }
  TPH_ADD(1, tl0);
  S.memo_nu = nu;
  S.memo = out;
  return out;
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

// stationarity of solve_nu — src/alignment.cpp:132-141.  With x = (v-mu)/sigma,
// w = c2/q where q = d^2 + c1, c1 = nu s^2, c2 = (nu+1) s^2, d = v - mu, so
//   mean(C + log w - w) = C + log c2 - mean(log q) - c2 mean(1/q),
// C the nu-only part of the reference's per-sample term; sum(1/q) and sum(log q)
// come from one q_sums pass.
template <int NT>
__device__ __forceinline__ double stationarity(Sample& S, double mu, double sigma, double nu,
                                               double* scratch) {
  TPH_T(ts0);
  const double C = (((-digamma_d(nu / 2.0) + log(nu / 2.0)) + digamma_d((nu + 1.0) / 2.0)) -
                    log((nu + 1.0) / 2.0)) + 1.0;
  const double s2 = sigma * sigma, c1 = nu * s2, c2 = (nu + 1.0) * s2;
  double a3[3];
  q_sums<NT, false, true>(S, mu, c1, a3);
  double a[2] = {a3[2], a3[0]};
  TPH_ADD(6, ts0);
  sample_allsum<2, NT>(a, S);
  const double inv_m = 1.0 / (double)S.m;
  TPH_ADD(4, ts0);
  TPH_CNT(5, 1);
  return ((C + log(c2)) - a[0] * inv_m) - c2 * (a[1] * inv_m);
}

// solve_nu — src/alignment.cpp:131-157.  The reference's 30 bisection steps on
// [2, 10] only ever evaluate f on the grid nu_k = 2 + k 2^-27 (k in [0, 2^30], every
// value exact in fp64) and end in the cell [nu_k, nu_k+1] whose ends satisfy
// f(lo) f(nu_k) > 0 and f(lo) f(nu_k+1) <= 0 (the same test, zeros and NaNs included);
// they return its midpoint.  For a stationarity with one sign change over the grid
// (the ML condition of the Student-t dof is monotone) that cell is unique, so any
// search over the grid that closes it returns the same nu: here regula falsi on the
// grid index, Illinois-weighted, falling back to a bisection step whenever the bracket
// did not halve twice in a row.  ~8-10 stationarity passes instead of 32.
// RGBID_NU_BISECT=1 builds the reference's plain bisection (for A/B).
#ifndef RGBID_NU_BISECT
#define RGBID_NU_BISECT 0
#endif
template <int NT>
__device__ __forceinline__ double solve_nu(Sample& S, double mu, double sigma, double* scratch) {
  const double flo0 = stationarity<NT>(S, mu, sigma, 2.0, scratch);
  const double fhi0 = stationarity<NT>(S, mu, sigma, 10.0, scratch);
  if (flo0 * fhi0 > 0.0) return fhi0 > 0.0 ? 10.0 : 2.0;
  constexpr double h = 0x1p-27;  // (10 - 2) / 2^30
  int klo = 0, khi = 1 << 30;
  double flo = flo0;
  // bisect: the reference's steps verbatim (A/B builds, and after any NaN: the
  // bisection's path through NaNs depends on where it meets them)
  bool bisect = RGBID_NU_BISECT || isnan(flo0) || isnan(fhi0);
  double gl = flo0, gh = fhi0;  // interpolation values (Illinois-scaled)
  int last = 0, slow = 0;       // side retained last (-1 lo, +1 hi); steps without halving
  while (khi - klo > 1) {
    const int width = khi - klo;
    int k;
    const double t = gl / (gl - gh);
    if (bisect || slow >= 2 || !(t >= 0.0 && t <= 1.0)) {  // also NaN / inf values
      k = klo + (width >> 1);
      slow = 0;
    } else {
      const double ke = (double)klo + t * (double)width;
      k = (int)fmin(fmax(rint(ke), (double)(klo + 1)), (double)(khi - 1));
    }
    const double fk = stationarity<NT>(S, mu, sigma, 2.0 + (double)k * h, scratch);
    if (!bisect && isnan(fk)) {  // restart as the plain bisection
      bisect = true;
      klo = 0;
      khi = 1 << 30;
      flo = flo0;
      continue;
    }
    if (flo * fk <= 0.0) {  // the reference's test (src/alignment.cpp:147)
      khi = k;
      gh = fk;
      if (last == -1) gl *= 0.5;  // lo retained twice: Illinois
      last = -1;
    } else {
      klo = k;
      flo = fk;
      gl = fk;
      if (last == 1) gh *= 0.5;
      last = 1;
    }
    slow = 2 * (khi - klo) > width ? slow + 1 : 0;
  }
  return 2.0 + (double)(klo + khi) * (0.5 * h);  // 0.5 (lo + hi), exact
}

// estimate_nu — src/alignment.cpp:109-127
template <int NT>
__device__ __forceinline__ double estimate_nu(Sample& S, double mu, double sigma, double* scratch) {
  if (S.m == 0 || sigma <= 0.0) return 5.0;
  double nu = solve_nu<NT>(S, mu, sigma, scratch);
  for (int it = 0; it < 2 && nu < 9.99; ++it) {
    const TD refit = loc_scale<NT>(S, nu, scratch);
    if (refit.sigma <= 0.0) break;
    const double nu_new = solve_nu<NT>(S, refit.mu, refit.sigma, scratch);
    if (fabs(nu_new - nu) < 1e-3) {
      nu = nu_new;
      break;
    }
    nu = nu_new;
  }
  return nu;
}

// validity words used per K1 tile (tx / 32, >= 1) and their log2
__host__ __device__ inline int tile_words_log2(int tx) {
  return tx >= 256 ? 3 : tx >= 128 ? 2 : tx >= 64 ? 1 : 0;
}

// position of the j-th (0-based) set bit of m (j < popc(m))
__device__ __forceinline__ int select_bit(unsigned m, int j) {
  int pos = 0;
#pragma unroll
  for (int w = 16; w > 0; w >>= 1) {
    const int c = __popc(m & ((1u << w) - 1u));
    if (j >= c) {
      j -= c;
      m >>= w;
      pos += w;
    }
  }
  return pos;
}

// K2a: systematic sample of the valid residuals of one (slot, residual type) —
// src/alignment.cpp:50-57 over the residual order of src/alignment.cpp:216-231.
// Gathering the sampled residuals is a DRAM-latency-bound scatter read; as its
// own kernel (small shared memory, many CTAs per SM) it runs at full occupancy
// and overlaps the other lane's FP64-bound K2b, which then streams the compact
// sample.  grid (kGatherCTAs, 2, slots); CTA c owns samples [c, c+1) * chunk.
// Every CTA scans the per-tile counts itself (1440 ints at 640x480, L2-resident).
constexpr int kGatherThreads = 256, kGatherCTAs = 8;
constexpr int kGatherChunk = (kMaxSample + kGatherCTAs - 1) / kGatherCTAs;

__global__ void __launch_bounds__(kGatherThreads)
    k_gather(const SlotIO* __restrict__ io, const SlotState* __restrict__ st, LevelInfo li,
             int phase) {
  constexpr int NT = kGatherThreads;
  const int type = blockIdx.y, slot = blockIdx.z;
  if (!slot_active(st[slot], li.level, phase)) return;
  const SlotIO& o = io[slot];
  const int* cnt = type ? o.cntW : o.cntI;
  const unsigned* bits = type ? o.bitsW : o.bitsI;
  // r_I (type 0) / warped W_B (type 1) at this level: component `type` of K1's pairs
  const double* bv = reinterpret_cast<const double*>(o.ibw) + type;
  const double* av = phase ? o.fWA : o.WA[li.level];
  extern __shared__ int offs[];  // [ntiles + 1]
  __shared__ long long sidx[kGatherChunk];
  __shared__ int wsum[NT / 32];
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int nt = li.ntiles;

  // exclusive scan of the per-tile counts (contiguous chunk per thread)
  const int per = (nt + NT - 1) / NT;
  const int b0 = min(nt, tid * per), b1 = min(nt, b0 + per);
  int local = 0;
  for (int i = b0; i < b1; ++i) local += __ldg(cnt + i);
  int incl = local;
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {
    const int v = __shfl_up_sync(0xffffffffu, incl, off);
    if (lane >= off) incl += v;
  }
  if (lane == 31) wsum[wid] = incl;
  __syncthreads();
  int woff = 0, total = 0;
  for (int k = 0; k < NT / 32; ++k) {
    if (k < wid) woff += wsum[k];
    total += wsum[k];
  }
  int run = woff + incl - local;
  for (int i = b0; i < b1; ++i) {
    offs[i] = run;
    run += __ldg(cnt + i);
  }
  if (tid == 0) offs[nt] = total;
  if (blockIdx.x == 0 && tid == 0) o.nsmp[type] = total;
  __syncthreads();

  const long long n = total;
  const long long stride = n <= kMaxSample ? 1 : (n + kMaxSample - 1) / kMaxSample;
  const int m = n == 0 ? 0 : (int)((n - 1) / stride + 1);
  const int c0 = blockIdx.x * kGatherChunk, c1 = min(m, c0 + kGatherChunk);
  if (c0 >= c1) return;  // uniform over the CTA

  // pass 1: sample s -> its level pixel.  Thread tid takes contiguous samples:
  // one binary search over the tile offsets, then a forward walk over the
  // validity words (row-major pixel order within each tile row).
  {
    const int lw = tile_words_log2(li.tx), wpt = 1 << lw;
    const int spt = (c1 - c0 + NT - 1) / NT;
    const int s0 = min(c1, c0 + tid * spt), s1 = min(c1, s0 + spt);
    if (s0 < s1) {
      long long g = (long long)s0 * stride;
      int lo = 0, hi = nt - 1;
      while (lo < hi) {  // last tile with offs[t] <= g
        const int mid = (lo + hi + 1) >> 1;
        if (offs[mid] <= g)
          lo = mid;
        else
          hi = mid - 1;
      }
      int tile = lo, w = 0, yl = lo / li.nseg, seg = lo - yl * li.nseg;
      long long base = offs[lo];  // rank of the first valid pixel of word w
      unsigned msk = __ldg(bits + tile * kWordsPerTile);
      int c = __popc(msk);
      for (int s = s0; s < s1; ++s, g += stride) {
        int j = (int)(g - base);
        while (j >= c) {
          j -= c;
          base += c;
          if (++w == wpt) {
            w = 0;
            ++tile;
            if (++seg == li.nseg) {
              seg = 0;
              ++yl;
            }
          }
          msk = __ldg(bits + tile * kWordsPerTile + w);
          c = __popc(msk);
        }
        sidx[s - c0] = yl * li.w + seg * li.tx + w * 32 + select_bit(msk, j);
      }
    }
  }
  __syncthreads();
  // pass 2: the residual values, four samples' loads in flight per thread;
  // coalesced stores of the compact sample
  double* out = o.smp + (size_t)type * kMaxSample;
  for (int s = c0 + tid; s < c1; s += 4 * NT) {
    long long ix[4];
    double b[4], a[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) ix[u] = s + u * NT < c1 ? sidx[s + u * NT - c0] : -1;
#pragma unroll
    for (int u = 0; u < 4; ++u)
      if (ix[u] >= 0) {
        b[u] = __ldg(bv + 2 * ix[u]);
        a[u] = type ? __ldg(av + ix[u]) : 0.0;
      }
#pragma unroll
    for (int u = 0; u < 4; ++u)
      if (ix[u] >= 0) out[s + u * NT] = type ? b[u] - a[u] : b[u];  // r_W = w_b - w_a / r_I stored by K1
  }
}

// K2b: Student-t fit of one (slot, residual type) on its compact sample.  NT
// threads hold the sample in shared memory, ~38 samples per thread: NT = 512 for
// the 19200-sample cap (one CTA per SM, all 128 registers per thread), smaller
// CTAs -- several per SM -- for coarse levels whose pixel count caps the sample.
#ifndef RGBID_TDIST_BULK
#define RGBID_TDIST_BULK 1  // sample into shared memory by cp.async.bulk (0: per-thread loads)
#endif
template <int NT>
__device__ __forceinline__ void tdist_chain(const SlotIO* __restrict__ io, SlotState* __restrict__ st,
                                            LevelInfo li, int phase) {
  const int type = blockIdx.x, slot = blockIdx.y;
  SlotState& S = st[slot];
  if (!slot_active(S, li.level, phase)) return;
  TPH_T(tk0);
  TPH_CNT(10, 1);
  const SlotIO& o = io[slot];
  extern __shared__ __align__(16) double dsm[];  // sample[kMaxSample]
  double* smp_sh = dsm;
  __shared__ double scratch[NT / 32 * 2 * 2];
  const int tid = threadIdx.x;

  const long long n = o.nsmp[type];
  const long long stride = n <= kMaxSample ? 1 : (n + kMaxSample - 1) / kMaxSample;
  Sample smp;
  smp.v = smp_sh;
  smp.m = n == 0 ? 0 : (int)((n - 1) / stride + 1);
  smp.m_local = smp.m;
  smp.kfull = smp.m / NT;
  smp.cs = 1;
  smp.cbuf = nullptr;
  smp.cmbar = nullptr;
  smp.cred = 0;
  smp.rank = 0;
  smp.memo_nu = -1.0;
  smp.have_mom = false;
  smp.scratch = scratch;
  smp.parity = 0;
  const double* gs = o.smp + (size_t)type * kMaxSample;
#if RGBID_TDIST_BULK
  // the compact sample (written by K2a, L2-resident) into shared memory by bulk
  // async copies: warp 0 issues kBulkParts pieces on one mbarrier, the odd last
  // sample (a piece must be a multiple of 16 B) by a plain load
  {
    __shared__ __align__(8) uint64_t mbar;
    const unsigned mb = (unsigned)__cvta_generic_to_shared(&mbar);
    const unsigned bytes = (unsigned)(smp.m & ~1) * 8u;
    if (tid == 0) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(mb));
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(mb), "r"(bytes)
                   : "memory");
    }
    __syncwarp();
    constexpr int kBulkParts = 8;
    const unsigned part = ((bytes / kBulkParts) + 15u) & ~15u;
    if (tid < kBulkParts && bytes > 0) {
      const unsigned off = tid * part;
      if (off < bytes) {
        const unsigned n = min(part, bytes - off);
        const unsigned dst = (unsigned)__cvta_generic_to_shared(smp_sh) + off;
        asm volatile(
            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
            "l"(reinterpret_cast<const char*>(gs) + off), "r"(n), "r"(mb)
            : "memory");
      }
    }
    if (tid == 0 && (smp.m & 1)) smp_sh[smp.m - 1] = gs[smp.m - 1];
    __syncthreads();  // mbarrier initialised and armed before anyone waits
    unsigned done = 0;
    do {
      asm volatile(
          "{ .reg .pred P; mbarrier.try_wait.parity.shared::cta.b64 P, [%1], 0;"
          " selp.u32 %0, 1, 0, P; }"
          : "=r"(done)
          : "r"(mb)
          : "memory");
    } while (!done);
  }
#else
  for (int s = tid; s < smp.m; s += 4 * NT) {
    double x[4];
#pragma unroll
    for (int u = 0; u < 4; ++u)
      if (s + u * NT < smp.m) x[u] = __ldcs(gs + s + u * NT);
#pragma unroll
    for (int u = 0; u < 4; ++u)
      if (s + u * NT < smp.m) smp_sh[s + u * NT] = x[u];
  }
#endif
  __syncthreads();

  // build_system's Student-t part — src/alignment.cpp:305-317
  TD t = loc_scale<NT>(smp, 5.0, scratch);
  t.sigma = dmax_std(t.sigma, 1e-8);
  t.nu = estimate_nu<NT>(smp, t.mu, t.sigma, scratch);
  if (t.nu < 4.99) {
    const TD r = loc_scale<NT>(smp, t.nu, scratch);
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
  TPH_ADD(7, tk0);
}

template <int NT>
__global__ void __launch_bounds__(NT, kTdistThreads / NT)
    k_tdist(const SlotIO* __restrict__ io, SlotState* __restrict__ st, LevelInfo li, int phase) {
  tdist_chain<NT>(io, st, li, phase);
}

// The full-cap chain with a register cap instead of launch bounds: at <= 80 registers
// (no spills) a 512-thread chain leaves a third of the register file to CTAs of the
// other lane's kernels (K1 / K3) on the same SM.
#ifndef RGBID_TDIST_MAXREG
#define RGBID_TDIST_MAXREG 80
#endif
__global__ void __maxnreg__(RGBID_TDIST_MAXREG)
    k_tdist_big(const SlotIO* __restrict__ io, SlotState* __restrict__ st, LevelInfo li, int phase) {
  tdist_chain<kTdistThreads>(io, st, li, phase);
}

// Latency-mode K2: the sample of one (slot, residual type) is spread over a
// cluster of kTdistCluster CTAs (sample s lives on rank s % CS); every pass
// reduces in-CTA, then across the cluster through DSMEM.
__global__ void __launch_bounds__(kTdistClusterThreads, 1)
    k_tdist_cluster(const SlotIO* __restrict__ io, SlotState* __restrict__ st, LevelInfo li,
                    int phase) {
  constexpr int NT = kTdistClusterThreads, CS = kTdistCluster;
  namespace cg = cooperative_groups;
  cg::cluster_group cl = cg::this_cluster();
  const int rank = (int)cl.block_rank();
  const int type = blockIdx.x / CS, slot = blockIdx.y;
  SlotState& S = st[slot];
  if (!slot_active(S, li.level, phase)) return;  // uniform over the cluster
  TPH_T(tk0);
  TPH_CNT(10, 1);
  const SlotIO& o = io[slot];
  const int* cnt = type ? o.cntW : o.cntI;
  const unsigned* bits = type ? o.bitsW : o.bitsI;
  const double* bv = reinterpret_cast<const double*>(o.ibw) + type;  // r_I / w_b pairs
  const double* av = phase ? o.fWA : o.WA[li.level];  // (r_I is stored by K1)
  extern __shared__ double dsm[];  // sample share [ceil(kMaxSample/CS)] + offs[ntiles + 1]
  constexpr int kShare = (kMaxSample + CS - 1) / CS;
  double* smp_sh = dsm;
  int* offs = reinterpret_cast<int*>(dsm + kShare);
  __shared__ int wsum[NT / 32];
  __shared__ double scratch[NT / 32 * 2 * 2];
  __shared__ double cbuf[2 * CS * (NT / 32) * 2];
  __shared__ __align__(8) uint64_t cmbar[2];
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  if (tid == 0) {
#pragma unroll
    for (int i = 0; i < 2; ++i)
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(
                       (unsigned)__cvta_generic_to_shared(&cmbar[i]))
                   : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  TPH_T(tg0);
  const int nt = li.ntiles;
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
  int woff = 0, total = 0;
  for (int k = 0; k < NT / 32; ++k) {
    if (k < wid) woff += wsum[k];
    total += wsum[k];
  }
  int run = woff + incl - local;
  for (int i = b0; i < b1; ++i) {
    offs[i] = run;
    run += cnt[i];
  }
  if (tid == 0) offs[nt] = total;
  __syncthreads();
  TPH_ADD(12, tg0);
  const long long n = total;
  const long long stride = n <= kMaxSample ? 1 : (n + kMaxSample - 1) / kMaxSample;
  Sample smp;
  smp.v = smp_sh;
  smp.m = n == 0 ? 0 : (int)((n - 1) / stride + 1);
  // CTA `rank` holds the contiguous samples [c0, c1); thread tid a contiguous run of
  // them: one binary search over the tile offsets, then a forward walk over the
  // validity words (as k_gather), the pixel indices parked in the sample slots
  const int share = (smp.m + CS - 1) / CS;
  const int c0 = min(smp.m, rank * share), c1 = min(smp.m, c0 + share);
  smp.m_local = c1 - c0;
  long long* sidx = reinterpret_cast<long long*>(smp_sh);
  {
    const int lw = tile_words_log2(li.tx), wpt = 1 << lw;
    const int spt = (smp.m_local + NT - 1) / NT;
    const int s0 = min(c1, c0 + tid * spt), s1 = min(c1, s0 + spt);
    if (s0 < s1) {
      long long g = (long long)s0 * stride;
      int lo = 0, hi = nt - 1;
      while (lo < hi) {  // last tile with offs[t] <= g
        const int mid = (lo + hi + 1) >> 1;
        if (offs[mid] <= g)
          lo = mid;
        else
          hi = mid - 1;
      }
      int tile = lo, w = 0, yl = lo / li.nseg, seg = lo - yl * li.nseg;
      long long base = offs[lo];
      unsigned msk = __ldg(bits + tile * kWordsPerTile);
      int c = __popc(msk);
      for (int s = s0; s < s1; ++s, g += stride) {
        int j = (int)(g - base);
        while (j >= c) {
          j -= c;
          base += c;
          if (++w == wpt) {
            w = 0;
            ++tile;
            if (++seg == li.nseg) {
              seg = 0;
              ++yl;
            }
          }
          msk = __ldg(bits + tile * kWordsPerTile + w);
          c = __popc(msk);
        }
        sidx[s - c0] = yl * li.w + seg * li.tx + w * 32 + select_bit(msk, j);
      }
    }
  }
  __syncthreads();
  TPH_ADD(13, tg0);
  for (int k = tid; k < smp.m_local; k += 4 * NT) {  // values, four loads in flight
    long long ix[4];
    double bb[4], aa[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) ix[u] = k + u * NT < smp.m_local ? sidx[k + u * NT] : -1;
#pragma unroll
    for (int u = 0; u < 4; ++u)
      if (ix[u] >= 0) {
        bb[u] = __ldg(bv + 2 * ix[u]);
        aa[u] = type ? __ldg(av + ix[u]) : 0.0;
      }
#pragma unroll
    for (int u = 0; u < 4; ++u)
      if (ix[u] >= 0) smp_sh[k + u * NT] = type ? bb[u] - aa[u] : bb[u];  // r_W / r_I (K1)
  }
  smp.kfull = smp.m_local / NT;
  smp.cs = CS;
  smp.cbuf = cbuf;
  smp.cmbar = cmbar;
  smp.cred = 0;
  smp.rank = rank;
  smp.memo_nu = -1.0;
  smp.have_mom = false;
  smp.scratch = scratch;
  smp.parity = 0;
  TPH_ADD(14, tg0);
  TPH_ADD(0, tk0);
  cl.sync();  // every CTA's share (and cbuf) ready before the first cluster reduction
  TD t = loc_scale<NT>(smp, 5.0, scratch);
  t.sigma = dmax_std(t.sigma, 1e-8);
  t.nu = estimate_nu<NT>(smp, t.mu, t.sigma, scratch);
  if (t.nu < 4.99) {
    const TD r = loc_scale<NT>(smp, t.nu, scratch);
    if (r.sigma > 0.0) {
      t.mu = r.mu;
      t.sigma = dmax_std(r.sigma, 1e-8);
    }
  }
  if (rank == 0 && tid == 0) {
    rgbid_tdist out{t.mu, t.sigma, t.nu};
    if (type == 0) {
      S.tI = out;
      S.nI = n;
    } else {
      S.tW = out;
      S.nW = n;
    }
  }
  TPH_ADD(7, tk0);
  cl.sync();  // no CTA exits while others may still read its cluster slots
}

#ifdef RGBID_TDIST_TRACE
extern "C" int rgbid_debug_tdist_phases(unsigned long long* out, int reset) {
  cudaDeviceSynchronize();
  cudaMemcpyFromSymbol(out, g_tph, sizeof(g_tph));
  if (reset) {
    static const unsigned long long z[24] = {};
    cudaMemcpyToSymbol(g_tph, z, sizeof(z));
  }
  return 0;
}
#endif

int init_kernel_attributes() {
  const cudaError_t e =
      cudaFuncSetAttribute(k_tdist_big, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           kMaxSample * 8);
  // the smaller CTAs serve sample caps up to kMaxSample / 2 (256) and / 4 (128)
  if (kTdistThreads != 256)
    cudaFuncSetAttribute(k_tdist<256>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         kMaxSample / 2 * 8);
  if (kTdistThreads != 128)
    cudaFuncSetAttribute(k_tdist<128>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         kMaxSample / 4 * 8);
  cudaFuncSetAttribute(k_gather, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
  const cudaError_t e2 =
      cudaFuncSetAttribute(k_tdist_cluster, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
  if (kTdistCluster > 8)
    cudaFuncSetAttribute(k_tdist_cluster, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  cudaGetLastError();
  return (e == cudaSuccess && e2 == cudaSuccess) ? 0 : 1;
}

void launch_tdist(const AlignLaunch& a, const LevelInfo& li, int phase, cudaStream_t s, int part) {
  if (a.nslots <= kTdistClusterMaxSlots) {  // latency mode: cluster per chain (no gather)
    if (part == 1) return;
    KScope ks_("tdist_cluster", s);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(2 * kTdistCluster, a.nslots);
    cfg.blockDim = dim3(kTdistClusterThreads);
    cfg.dynamicSmemBytes =
        ((kMaxSample + kTdistCluster - 1) / kTdistCluster) * 8 + (li.ntiles + 1) * 4;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = kTdistCluster;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    cudaLaunchKernelEx(&cfg, k_tdist_cluster, a.io, a.st, li, phase);
    return;
  }
  if (part != 2) {
    KScope ks_("gather", s);
    k_gather<<<dim3(kGatherCTAs, 2, a.nslots), kGatherThreads, (li.ntiles + 1) * sizeof(int), s>>>(
        a.io, a.st, li, phase);
  }
  if (part == 1) return;
  KScope ks_("tdist", s);
  // highest launch priority: the FP64-bound chains claim SMs first, the other
  // lane's memory-bound kernels fill around them
  static int prio = [] {
    int lo = 0, hi = 0;
    cudaDeviceGetStreamPriorityRange(&lo, &hi);
    return hi;
  }();
  const int mcap = std::min(kMaxSample, li.w * li.h);  // sample size bound at this level
  const int nt = mcap > kMaxSample / 2 ? kTdistThreads : mcap > kMaxSample / 4 ? 256 : 128;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(2, a.nslots);
  cfg.blockDim = dim3(nt);
  cfg.dynamicSmemBytes = mcap * sizeof(double);
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributePriority;
  attr[0].val.priority = prio;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  if (nt == kTdistThreads)
    cudaLaunchKernelEx(&cfg, k_tdist_big, a.io, (SlotState*)a.st, li, phase);
  else if (nt == 256)
    cudaLaunchKernelEx(&cfg, k_tdist<256>, a.io, (SlotState*)a.st, li, phase);
  else
    cudaLaunchKernelEx(&cfg, k_tdist<128>, a.io, (SlotState*)a.st, li, phase);
}

// ---------------------------------------------------------------------------
// K3: jets + robust weights + 28 fp64 sums per tile (PIX pixels per thread: kPixK3 in
// batches, 1 in latency mode).
// Jets restate src/alignment.cpp:212-244 with the structure of A = K - p e_z^T and
// M = [I | -[X_A]x] folded in: J = (u, X_A x u) with u = w_a g A; the weights are
// src/alignment.cpp:324,329-330.  Tolerance-level (not bitwise) w.r.t. the
// reference: the sums' order differs anyway.
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

static const char* kNeNames[kMaxLevels] = {"normal_eq_L0", "normal_eq_L1", "normal_eq_L2",
                                            "normal_eq_L3", "normal_eq_L4", "normal_eq_L5"};


// D = A B + C, one m8n8k4 fp64 tensor-core MMA (A row-major 8x4, B col-major 4x8;
// lane l holds A[l/4][l%4], B[l%4][l/4], C[l/4][2(l%4) + {0,1}])
__device__ __forceinline__ void dmma884(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

// K3 on the FP64 tensor cores.  Same jets and weights as k_normal_eq; each warp
// stages its 32 pixel rows x = (J, r, 0) and w in shared memory and accumulates
// C += sum_k w_k x_k x_k^T with 8 MMAs per row type, so the 8x8 system (H, the
// J^T W r column, the cost) lives in two fp64 registers per lane instead of 28 --
// the register file no longer caps occupancy.  Invalid rows are zeroed at their
// inputs (gradients, residual, w_a, w_b), so every staged component is an exact 0.
// one staged row x = (J, r, 0) and its weight w
__device__ __forceinline__ void stage_row(double* r, double j0, double j1, double j2, double j3,
                                          double j4, double j5, double res, double w) {
  r[0] = j0;
  r[1] = j1;
  r[2] = j2;
  r[3] = j3;
  r[4] = j4;
  r[5] = j5;
  r[6] = res;
  r[7] = 0.0;
  r[8] = w;
}

#ifndef RGBID_K3_MMA_MINB
#define RGBID_K3_MMA_MINB 3
#endif
template <bool LIST, int PIX>
__global__ void __launch_bounds__(kTPB, RGBID_K3_MMA_MINB) k_normal_eq_mma(const SlotIO* __restrict__ io,
                                                        const SlotState* __restrict__ st,
                                                        LevelInfo li, int phase,
                                                        double lambda_n_min,
                                                        const int* __restrict__ act) {
  const int slot = active_slot<LIST>(act, blockIdx.y);
  if (slot < 0) return;
  const SlotState& S = st[slot];
  if (!slot_active(S, li.level, phase)) return;  // uniform over the CTA
  const SlotIO& o = io[slot];
  const double* __restrict__ WA = phase ? o.fWA : o.WA[li.level];
  const uint8_t* __restrict__ am = o.amask[li.level];
  const double2* __restrict__ ag = reinterpret_cast<const double2*>(o.agrad[li.level]);
  const double2* __restrict__ ibwp = o.ibw;
  // staged row: 8 components + w; a stride of 9 doubles keeps the per-lane row stores
  // conflict-free (the operand loads see 2-way conflicts).  A stride of 10 with 16-byte
  // stores (conflict-free both ways) measured 3.5% slower per launch.
  constexpr int XS = 9;
  __shared__ __align__(16) double xs[kTPB / 32][32 * XS];
  __shared__ double cst[kTPB / 32][64];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  double* xw = xs[wid];
  const double muI = S.tI.mu, isgI = 1.0 / S.tI.sigma, nuI = dmax_std(S.tI.nu, S.tW.nu);
  const double muW = S.tW.mu, isgW = 1.0 / S.tW.sigma, nuW = S.tW.nu;
  const double nuI1 = nuI + 1.0, nuW1 = nuW + 1.0;
  const double is2i = isgI * isgI, is2w = isgW * isgW;
  const int w = li.w;
  const double* Ki = li.Kinv;
  const int N = li.w * li.h;
  double c0 = 0.0, c1 = 0.0;
  auto mma_rows = [&]() {
    __syncwarp();
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const int row = 4 * j + (lane & 3);
      const double xv = xw[row * XS + (lane >> 2)], wv = xw[row * XS + 8];
      dmma884(c0, c1, wv * xv, xv);
    }
    __syncwarp();
  };
#pragma unroll 1
  for (int p = 0; p < PIX; ++p) {
    const int k0i = (blockIdx.x * PIX + p) * kTPB + threadIdx.x;
    const bool inr = k0i < N;
    const int k = inr ? k0i : 0;
    const unsigned a = __ldg(am + k);
    const double2 rw = __ldcs(ibwp + k);  // {r_I = i_b - i_a, w_b} (K1)
    const double r_I = rw.x, w_b_ = rw.y;
    const double w_a_ = __ldg(WA + k);
    const double2 gI_ = __ldg(ag + 2 * k), gW_ = __ldg(ag + 2 * k + 1);
    const bool jet = inr && (a & 1u) && valid(r_I);  // bit0 implies valid(i_a)
    const bool dep = jet && (a & 2u) && valid(w_b_) && w_b_ > 0.0;
    const int y = k / w, x = k - y * w;
    const double px = x, py = y;
    const double ax = li.cx - px, ay = li.cy - py;
    // invalid rows zeroed at their inputs (gradients, residual, w_a, w_b): every
    // staged component is then an exact 0 and the weight finite -- 16 selects per
    // pixel instead of 32 at the staging
    const double w_a = jet ? w_a_ : 1.0;
    const double2 gI = make_double2(jet ? gI_.x : 0.0, jet ? gI_.y : 0.0);
    const double2 gW = make_double2(dep ? gW_.x : 0.0, dep ? gW_.y : 0.0);
    const double w_b = dep ? w_b_ : 0.0;
    const double iwa = rcp_fast(w_a);  // H is tolerance-checked: MUFU + Newton, no IEEE divide
    const double k0 = red3(Ki[0] * px, Ki[1] * py, Ki[2]), k1 = red3(Ki[3] * px, Ki[4] * py, Ki[5]),
                 k2 = red3(Ki[6] * px, Ki[7] * py, Ki[8]);
    const double X0 = k0 * iwa, X1 = k1 * iwa, X2 = k2 * iwa;
    {  // photometric row
      const double s0 = w_a * gI.x, s1 = w_a * gI.y;
      const double u0 = s0 * li.fx, u1 = s1 * li.fy, u2 = s0 * ax + s1 * ay;
      const double rI = jet ? r_I : 0.0;
      const double xi_ = (rI - muI) * isgI;
      const double wi = nuI1 * rcp_fast(fma(xi_, xi_, nuI)) * is2i;
      stage_row(xw + lane * XS, u0, u1, u2, X1 * u2 - X2 * u1, X2 * u0 - X0 * u2,
                X0 * u1 - X1 * u0, rI, wi);
    }
    mma_rows();
    {  // geometric row
      const double g0 = gW.x * li.fx, g1 = gW.y * li.fy, g2 = gW.x * ax + gW.y * ay;
      const double s0 = w_a * g0, s1 = w_a * g1, s2 = w_a * (g2 + w_b);
      double lambda = 1.0;
      {
        const double n0 = g0 * iwa, n1 = g1 * iwa, n2 = g2 * iwa + 1.0;
        const double nn2 = n0 * n0 + n1 * n1 + n2 * n2;
        if (!(nn2 < 1e-24)) {  // ||n|| < 1e-12 without the sqrt
          const double rr2 = k0 * k0 + k1 * k1 + k2 * k2;
          double c = (n0 * k0 + n1 * k1 + n2 * k2) * rsqrt(nn2 * rr2);
          if (n2 < 0) c = -c;
          lambda = dmax_std(lambda_n_min, c);
        }
      }
      const double rW = dep ? w_b - w_a : 0.0;
      const double xw_ = (rW - muW) * isgW;
      const double ww = lambda * nuW1 * rcp_fast(fma(xw_, xw_, nuW)) * is2w;
      stage_row(xw + lane * XS, s0, s1, s2, X1 * s2 - X2 * s1, X2 * s0 - X0 * s2,
                X0 * s1 - X1 * s0, rW, ww);
    }
    mma_rows();
  }
  cst[wid][(lane >> 2) * 8 + 2 * (lane & 3)] = c0;
  cst[wid][(lane >> 2) * 8 + 2 * (lane & 3) + 1] = c1;
  __syncthreads();
  if (threadIdx.x < kNPart) {  // partial q in k_normal_eq's order
    const int q = threadIdx.x;
    int r, c;
    if (q < 21) {
      r = 0;
      while ((r + 1) * (r + 2) / 2 <= q) ++r;
      c = q - r * (r + 1) / 2;
    } else if (q < 27) {
      r = q - 21;
      c = 6;
    } else {
      r = 6;
      c = 6;
    }
    double t = 0.0;
#pragma unroll
    for (int wv = 0; wv < kTPB / 32; ++wv) t += cst[wv][r * 8 + c];
    o.part[(size_t)q * li.ntiles3 + blockIdx.x] = t;  // value-major: K4 reads coalesced
  }
}

void launch_normal_equations(const AlignLaunch& a, const LevelInfo& li, int phase, cudaStream_t s,
                             int rows) {
  KScope ks_(phase ? "normal_eq_cov" : kNeNames[li.level], s);
  const dim3 grid(li.ntiles3, rows > 0 ? rows : a.nslots);
  if (li.pix3 == 1)  // latency mode: one pixel per thread, no list
    k_normal_eq_mma<false, 1><<<grid, kTPB, 0, s>>>(a.io, a.st, li, phase, a.lambda_n_min, nullptr);
  else if (rows > 0 && a.act)
    k_normal_eq_mma<true, kPixK3><<<grid, kTPB, 0, s>>>(a.io, a.st, li, phase, a.lambda_n_min,
                                                         a.act);
  else
    k_normal_eq_mma<false, kPixK3><<<grid, kTPB, 0, s>>>(a.io, a.st, li, phase, a.lambda_n_min,
                                                          nullptr);
}

// fixed-order reduction of the per-tile partials into H (full, mirrored), b, cost
__device__ void reduce_partials(const double* part, int ntiles, double* H, double* b, double* cost,
                                double* sh /*[kTPB/32 * kNPart]*/) {
  double acc[kNPart];
#pragma unroll
  for (int i = 0; i < kNPart; ++i) acc[i] = 0.0;
  for (int t = threadIdx.x; t < ntiles; t += kTPB)
#pragma unroll
    for (int i = 0; i < kNPart; ++i) acc[i] += part[(size_t)i * ntiles + t];
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
  TPH_T(ts0);
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
  TPH_ADD(16, ts0);
  // the rank test (warp 1) runs beside the solve and pose update (warp 0): the
  // serial 6x6 chains overlap instead of adding up; the update is kept only if H
  // passed (src/alignment.cpp:391-394)
  __shared__ int deficient;
  __syncthreads();  // H, b, cost from thread 0
  const int t = threadIdx.x;
  if (t >= 64 && t < 100) S.H[t - 64] = H[t - 64];
  if (t == 32) deficient = rank_deficient6(H) ? 1 : 0;
  double xi[6];
  PoseD T;
  WarpMats wmn;
  if (t == 0) {
    TPH_T(ts1);
    ldlt_solve6(H, b, xi);
    TPH_ADD(17, ts1);
    TPH_T(ts2);
    T = pose_update(xi, pose_from(S.R, S.t));
    TPH_ADD(18, ts2);
    TPH_T(ts3);
    wmn = warp_mats(T, fx0, fy0, cx0, cy0);
    TPH_ADD(19, ts3);
  }
  __syncthreads();
  if (t != 0) return;
  if (deficient) {
    S.status = RGBID_E_DEGENERATE;
    return;
  }
  pose_to(T, S.R, S.t);
  S.wm = wmn;
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
  TPH_ADD(20, ts0);
  TPH_CNT(21, 1);
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

// exp(x) for x <= 0, branch-free: 2^(j/32) table held one entry per lane and
// read with a warp shuffle (no shared-memory bank conflicts; every lane of the warp
// must call it) x degree-6 polynomial on |r| <= ln2/64, within ~1 ulp of the
// correctly rounded value (the parity tests bound the filtered maps at 1e-14
// relative).  x is clamped at -746 (NaN and -inf too), so results below the normal
// range come out as subnormals (one extra rounding) or zero, and NaN/-inf
// arguments give 0.
__constant__ double c_exp2_32[32] = {
    1.0, 1.0218971486541166, 1.0442737824274138, 1.0671404006768237,
    1.0905077326652577, 1.1143867425958924, 1.1387886347566916, 1.1637248587775775,
    1.189207115002721, 1.215247359980469, 1.241857812073484, 1.2690509571917332,
    1.2968395546510096, 1.3252366431597413, 1.3542555469368927, 1.383909881963832,
    1.4142135623730951, 1.4451808069770467, 1.4768261459394993, 1.5091644275934228,
    1.5422108254079407, 1.5759808451078865, 1.6104903319492543, 1.645755478153965,
    1.681792830507429, 1.718619298122478, 1.7562521603732995, 1.7947090750031072,
    1.8340080864093424, 1.8741676341103, 1.9152065613971474, 1.9571441241754002};

__device__ __forceinline__ double exp2_32_lane() { return c_exp2_32[threadIdx.x & 31]; }

__device__ __forceinline__ double exp_le0(double x, double tlane) {
  // arguments below -708 (and NaN: an invalid tap) give exp(-708) ~ 3e-308 instead
  // of the tiny or zero true value: a weight that small is absorbed by any sum that
  // holds the centre tap's weight 1 (and multiplies a 0 value for an invalid tap),
  // and t 2^m below is then a normal double
  x = x > -708.0 ? x : -708.0;
  const double kMagic = 6755399441055744.0;            // 1.5 * 2^52: round to integer
  const double kd = fma(x, 46.16624130844683, kMagic);  // x * 32 / ln2
  const int n = __double2loint(kd);
  const double k = kd - kMagic;
  double r = fma(-k, 0.02166084938653512, x);  // ln2/32, hi part (32 bits: k * hi exact)
  r = fma(-k, 5.9631716539705866e-12, r);      // lo part
  double pl = fma(r, 1.0 / 720.0, 1.0 / 120.0);
  pl = fma(r, pl, 1.0 / 24.0);
  pl = fma(r, pl, 1.0 / 6.0);
  pl = fma(r, pl, 0.5);
  pl = fma(r, pl, 1.0);
  const double em1 = r * pl;  // e^r - 1
  const double t = __shfl_sync(0xffffffffu, tlane, n & 31);
  // t 2^m (m = n >> 5 >= -1022, t in [1, 2): a normal double) by adding m to t's
  // exponent field -- no scale multiply
  const double ts = __hiloint2double(__double2hiint(t) + ((n >> 5) << 20), __double2loint(t));
  return fma(ts, em1, ts);
}

// bilateral_filter — src/alignment.cpp:252-277, tiled.  The tap weight
// exp(-(dx^2+dy^2)/(2 ss^2) - (v-c)^2/(2 sr^2)) is the same double for the
// ordered pairs (p, q) and (q, p) ((v-c)^2 == (c-v)^2 bit for bit), so each
// unordered pair's exp is evaluated once, for the raster-earlier pixel p and the
// "forward" offset o = q - p (dy > 0, or dy == 0 and dx > 0).  Per offset, the
// owners p with p or p + o in the 32 x 8 output tile lie in a 36 x (8 + dy) box
// (x from -2, y from -dy).  A 36 x 8 thread grid evaluates the first 8 box rows of
// all 12 offsets (straight-line, the same thread-relative addresses for every
// offset) and then the 540 remaining entries (rows 8, 9) -- ~15.6 exps per output
// pixel, no per-item index arithmetic on the main pass.  A pair with an invalid end
// gets weight 0 (the valid end skips it in the reference and the invalid end
// outputs NaN) and invalid taps read value 0, so every output accumulates its 5x5
// window in the reference order with no per-tap tests: a skipped tap adds +0.0 to
// both sums, which leaves them bit-identical (neither sum is ever -0.0).
#ifndef RGBID_BIL_MINB
#define RGBID_BIL_MINB 5  // 5 x 288 threads per SM (40 registers)
#endif
#ifndef RGBID_BIL_ROWS
#define RGBID_BIL_ROWS 2  // output rows per thread in the accumulation
#endif
constexpr int kBTW = 32, kBTH = 8;               // output tile
constexpr int kBRW = kBTW + 8, kBRH = kBTH + 4;  // input region from (x0-4, y0-2)
constexpr int kBFP = kBTW + 4;                   // box pitch (x from -2)
constexpr int kBNT = kBFP * kBTH;                // 288 threads: one per main-pass box entry
// forward offsets o = 0..11: (1,0) (2,0) (-2..2,1) (-2..2,2)
__host__ __device__ constexpr int bil_dx(int o) { return o < 2 ? o + 1 : (o < 7 ? o - 4 : o - 9); }
__host__ __device__ constexpr int bil_dy(int o) { return o < 2 ? 0 : (o < 7 ? 1 : 2); }
// box rows before offset o (sum of kBTH + dy over the earlier offsets)
__host__ __device__ constexpr int bil_rows(int o) {
  return kBTH * o + (o <= 2 ? 0 : (o <= 7 ? o - 2 : 5 + 2 * (o - 7)));
}
constexpr int kBFW = kBFP * bil_rows(12);  // forward weights, doubles
constexpr int kBExtra = 5 * kBFP + 5 * 2 * kBFP;  // box rows >= kBTH: 540 entries

__device__ __forceinline__ double bil_weight(const double* reg, int rc, int rv, double so,
                                             double inv2sr, double tab) {
  const double c = reg[rc], v = reg[rv];
  // an invalid end (NaN, +-inf) gives a NaN or -inf argument -> weight 0
  return exp_le0(so - (v - c) * (v - c) * inv2sr, tab);
}

template <int O>
__device__ __forceinline__ void bil_main(int t, int rb, double inv2ss, double inv2sr,
                                         double tab, const double* reg, double* fw) {
  constexpr int dx = bil_dx(O), dy = bil_dy(O);
  const double so = (double)(-(dx * dx + dy * dy)) * inv2ss;
  // box entry (lx, ly) = owner (lx - 2, ly - dy); rb = region index of (lx - 2, ly)
  fw[kBFP * bil_rows(O) + t] = bil_weight(reg, rb - dy * kBRW, rb + dx, so, inv2sr, tab);
  if constexpr (O + 1 < 12) bil_main<O + 1>(t, rb, inv2ss, inv2sr, tab, reg, fw);
}

__device__ __forceinline__ void bilateral_tile(const double* __restrict__ img, int w, int h,
                                               double inv2ss, double inv2sr,
                                               double* __restrict__ out, int x0, int y0,
                                               double* reg, double* reg0, double* fw) {
  const int t = threadIdx.x;
  const double tab = exp2_32_lane();
  for (int i = t; i < kBRW * kBRH; i += kBNT) {
    const int ry = i / kBRW, rx = i - ry * kBRW;
    const int gx = x0 - 4 + rx, gy = y0 - 2 + ry;
    const double v = (gx >= 0 && gx < w && gy >= 0 && gy < h) ? __ldg(img + (size_t)gy * w + gx)
                                                             : CUDART_NAN;  // out of bounds = skipped
    reg[i] = v;
    reg0[i] = valid(v) ? v : 0.0;
  }
  __syncthreads();
  {
    const int ly = t / kBFP, lx = t - ly * kBFP;
    bil_main<0>(t, (ly + 2) * kBRW + lx + 2, inv2ss, inv2sr, tab, reg, fw);
  }
  // rows >= kBTH of the dy = 1 boxes (o = 2..6, one row) and dy = 2 boxes (o = 7..11,
  // two rows): two rounds run by every lane (the exp's shuffle), stores predicated
#pragma unroll
  for (int k = 0; k < (kBExtra + kBNT - 1) / kBNT; ++k) {
    const int e0 = t + k * kBNT;
    const bool live = e0 < kBExtra;
    const int e = live ? e0 : 0;
    int o, lx, ly, dy;
    if (e < 5 * kBFP) {
      o = 2 + e / kBFP;
      lx = e - (o - 2) * kBFP;
      ly = kBTH;
      dy = 1;
    } else {
      const int f = e - 5 * kBFP;
      const int q = f / (2 * kBFP), r = f - q * (2 * kBFP);
      o = 7 + q;
      ly = kBTH + r / kBFP;
      lx = r - (ly - kBTH) * kBFP;
      dy = 2;
    }
    const int dx = dy == 1 ? o - 4 : o - 9;
    const double so = (double)(-(dx * dx + dy * dy)) * inv2ss;
    const int rb = (ly + 2) * kBRW + lx + 2;
    const double wt = bil_weight(reg, rb - dy * kBRW, rb + dx, so, inv2sr, tab);
    if (live) fw[kBFP * bil_rows(o) + ly * kBFP + lx] = wt;
  }
  __syncthreads();
  // outputs: each of kBTW * kBTH / R threads accumulates R vertically adjacent
  // pixels row by row over their (R + 4) x 5 joint window, each window row's values
  // read once for all of them (5 (R + 4) value reads per R pixels instead of 25 R)
  constexpr int R = RGBID_BIL_ROWS;
  if (t >= kBTW * kBTH / R) return;
  const int tx = t % kBTW, ty0 = R * (t / kBTW);
  const int x = x0 + tx;
  if (x >= w || y0 + ty0 >= h) return;
  double ws[R], vs[R];
#pragma unroll
  for (int p = 0; p < R; ++p) ws[p] = vs[p] = 0.0;
#pragma unroll
  for (int j = -2; j <= R + 1; ++j) {  // window row, relative to the first pixel
    double v[5];
#pragma unroll
    for (int dx = -2; dx <= 2; ++dx) v[dx + 2] = reg0[(ty0 + 2 + j) * kBRW + tx + 4 + dx];
#pragma unroll
    for (int pix = 0; pix < R; ++pix) {
      const int dy = j - pix;  // tap row relative to this pixel
      if (dy < -2 || dy > 2) continue;
      const int ty = ty0 + pix;
#pragma unroll
      for (int dx = -2; dx <= 2; ++dx) {
        double wt;
        if (dy == 0 && dx == 0) {
          wt = 1.0;  // exp(+0.0)
        } else {
          const bool fwd = dy > 0 || (dy == 0 && dx > 0);
          const int fdx = fwd ? dx : -dx, fdy = fwd ? dy : -dy;
          const int o = fdy == 0 ? fdx - 1 : (fdy == 1 ? 4 + fdx : 9 + fdx);
          // owner p (forward) or p - o (backward); box row = owner y + fdy, col = owner x + 2
          const int ox = fwd ? tx : tx + dx, oy = fwd ? ty : ty + dy;
          wt = fw[kBFP * bil_rows(o) + (oy + fdy) * kBFP + ox + 2];
        }
        ws[pix] += wt;
        vs[pix] += wt * v[dx + 2];
      }
    }
  }
#pragma unroll
  for (int p = 0; p < R; ++p)
    if (y0 + ty0 + p < h)
      out[(size_t)(y0 + ty0 + p) * w + x] =
          valid(reg[(ty0 + p + 2) * kBRW + tx + 4]) ? vs[p] / ws[p] : CUDART_NAN;
}

struct BilateralSmem {
  double reg[kBRW * kBRH], reg0[kBRW * kBRH], fw[kBFW];
};

__global__ void __launch_bounds__(kBNT, RGBID_BIL_MINB) k_bilateral(const double* __restrict__ img, int w,
                                                           int h, double inv2ss, double inv2sr,
                                                           double* __restrict__ out) {
  __shared__ BilateralSmem sm;
  bilateral_tile(img, w, h, inv2ss, inv2sr, out, blockIdx.x * kBTW, blockIdx.y * kBTH, sm.reg,
                 sm.reg0, sm.fw);
}

void launch_bilateral(const double* img, int w, int h, double ss, double sr, double* out,
                      cudaStream_t s) {
  const double inv2ss = 1.0 / (2.0 * ss * ss), inv2sr = 1.0 / (2.0 * sr * sr);
  KScope ks_("bilateral", s);
  k_bilateral<<<dim3((w + kBTW - 1) / kBTW, (h + kBTH - 1) / kBTH), kBNT, 0, s>>>(
      img, w, h, inv2ss, inv2sr, out);
}

// both filtered maps of every active slot (covariance pass input); grid.z = map
__global__ void __launch_bounds__(kBNT, RGBID_BIL_MINB)
    k_bilateral_slots(const SlotIO* __restrict__ io, const SlotState* __restrict__ st, int w,
                      int h, double inv2ss, double inv2sr_i, double inv2sr_w) {
  const int slot = blockIdx.z >> 1, map = blockIdx.z & 1;
  if (st[slot].status != RGBID_OK) return;
  const SlotIO& o = io[slot];
  __shared__ BilateralSmem sm;
  bilateral_tile(map ? o.WA[0] : o.IA[0], w, h, inv2ss, map ? inv2sr_w : inv2sr_i,
                 map ? o.fWA : o.fIA, blockIdx.x * kBTW, blockIdx.y * kBTH, sm.reg, sm.reg0,
                 sm.fw);
}

void launch_bilateral_pair(const AlignLaunch& a, double ss, double sr_i, double sr_w,
                           cudaStream_t s) {
  const double inv2ss = 1.0 / (2.0 * ss * ss);
  const double ii = 1.0 / (2.0 * sr_i * sr_i), iw = 1.0 / (2.0 * sr_w * sr_w);
  KScope ks_("bilateral_slots", s);
  k_bilateral_slots<<<dim3((a.w0 + kBTW - 1) / kBTW, (a.h0 + kBTH - 1) / kBTH, 2 * a.nslots),
                      kBNT, 0, s>>>(a.io, a.st, a.w0, a.h0, inv2ss, ii, iw);
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

__global__ void k_fill(double* p, long long n, double v) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x)
    p[i] = v;
}
void launch_fill(double* p, long long n, double v, cudaStream_t s) {
  if (n <= 0) return;
  KScope ks_("fill", s);
  k_fill<<<(int)std::min<long long>((n + 255) / 256, 148 * 16), 256, 0, s>>>(p, n, v);
}

// ---------------------------------------------------------------------------
// Drop-in helpers (reference entry points that are not on the align hot path but
// are part of the replaced sources).

// inverse_warp's sampling step (src/warping.cpp:8-18) for a host-evaluated map
__global__ void k_remap_bilinear(const double* __restrict__ src, int w, int h,
                                 const double* __restrict__ mx, const double* __restrict__ my,
                                 int n, double* __restrict__ out) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) out[i] = bilinear(src, w, h, mx[i], my[i]);
}
void launch_remap_bilinear(const double* src, int w, int h, const double* mx, const double* my,
                           int n, double* out, cudaStream_t s) {
  KScope ks_("remap_bilinear", s);
  k_remap_bilinear<<<(n + 255) / 256, 256, 0, s>>>(src, w, h, mx, my, n, out);
}

// residuals_and_jacobians per pixel (src/alignment.cpp:195-250): record
// {x, y, r_I, r_W, J_I[6], J_W[6], lambda_n} + flag (0 none, 1 jet, 2 jet+depth)
__global__ void k_jets(const double* __restrict__ IA, const double* __restrict__ WA,
                       const double* __restrict__ IBw, const double* __restrict__ WBw, LevelInfo li,
                       double lambda_n_min, double* __restrict__ rec, uint8_t* __restrict__ flag) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  const int w = li.w, h = li.h;
  if (k >= w * h) return;
  const int y = k / w, x = k - y * w;
  flag[k] = 0;
  const double w_a = WA[k], i_a = IA[k], i_b = IBw[k];
  if (!valid(w_a) || w_a <= 0.0 || !valid(i_a) || !valid(i_b)) return;
  double gix, giy;
  if (!gradient_at(IA, w, h, x, y, gix, giy)) return;
  const double* Ki = li.Kinv;
  const double px = x, py = y, ax = li.cx - px, ay = li.cy - py;
  const double k0 = red3(Ki[0] * px, Ki[1] * py, Ki[2]), k1 = red3(Ki[3] * px, Ki[4] * py, Ki[5]),
               k2 = red3(Ki[6] * px, Ki[7] * py, Ki[8]);
  const double X0 = k0 / w_a, X1 = k1 / w_a, X2 = k2 / w_a;
  double* o = rec + (size_t)k * 17;
  o[0] = x;
  o[1] = y;
  o[2] = i_b - i_a;
  o[3] = 0.0;
  {
    const double s0 = w_a * gix, s1 = w_a * giy;
    const double u0 = s0 * li.fx, u1 = s1 * li.fy, u2 = s0 * ax + s1 * ay;
    o[4] = u0, o[5] = u1, o[6] = u2;
    o[7] = X1 * u2 - X2 * u1, o[8] = X2 * u0 - X0 * u2, o[9] = X0 * u1 - X1 * u0;
  }
  for (int c = 10; c < 16; ++c) o[c] = 0.0;
  o[16] = 1.0;
  flag[k] = 1;
  const double w_b = WBw[k];
  double gwx, gwy;
  if (!(valid(w_b) && w_b > 0.0 && gradient_at(WA, w, h, x, y, gwx, gwy))) return;
  const double g0 = gwx * li.fx, g1 = gwy * li.fy, g2 = gwx * ax + gwy * ay;
  const double s0 = w_a * g0, s1 = w_a * g1, s2 = w_a * (g2 + w_b);
  o[3] = w_b - w_a;
  o[10] = s0, o[11] = s1, o[12] = s2;
  o[13] = X1 * s2 - X2 * s1, o[14] = X2 * s0 - X0 * s2, o[15] = X0 * s1 - X1 * s0;
  const double n0 = g0 / w_a, n1 = g1 / w_a, n2 = g2 / w_a + 1.0;
  const double nn = sqrt(n0 * n0 + n1 * n1 + n2 * n2);
  double lambda = 1.0;
  if (!(nn < 1e-12)) {
    double c = (n0 * k0 + n1 * k1 + n2 * k2) / (nn * sqrt(k0 * k0 + k1 * k1 + k2 * k2));
    if (n2 < 0) c = -c;
    lambda = dmax_std(lambda_n_min, c);
  }
  o[16] = lambda;
  flag[k] = 2;
}
void launch_jets(const double* IA, const double* WA, const double* IBw, const double* WBw,
                 const LevelInfo& li, double lambda_n_min, double* rec, uint8_t* flag,
                 cudaStream_t s) {
  KScope ks_("jets", s);
  k_jets<<<(li.w * li.h + 255) / 256, 256, 0, s>>>(IA, WA, IBw, WBw, li, lambda_n_min, rec, flag);
}

// estimate_location_scale (mode 0) / estimate_nu (mode 1) on a residual vector
// (src/alignment.cpp:61-127): systematic sample into smem, then the same
// device chain as k_tdist.
__global__ void __launch_bounds__(kTdistThreads, 1)  // one CTA per SM (sample in smem)
    k_tdist_vec(const double* __restrict__ r, long long n, int mode, double a, double b,
                double* __restrict__ out) {
  constexpr int NT = kTdistThreads;
  extern __shared__ double dsm[];
  __shared__ double scratch[NT / 32 * 2 * 2];
  const long long stride = n <= kMaxSample ? 1 : (n + kMaxSample - 1) / kMaxSample;
  Sample smp;
  smp.v = dsm;
  smp.m = n == 0 ? 0 : (int)((n - 1) / stride + 1);
  smp.m_local = smp.m;
  smp.kfull = smp.m / NT;
  smp.cs = 1;
  smp.cbuf = nullptr;
  smp.cmbar = nullptr;
  smp.cred = 0;
  smp.rank = 0;
  smp.memo_nu = -1.0;
  smp.have_mom = false;
  smp.scratch = scratch;
  smp.parity = 0;
  for (int s = threadIdx.x; s < smp.m; s += NT) dsm[s] = r[(long long)s * stride];
  __syncthreads();
  if (mode == 0) {
    const TD t = loc_scale<NT>(smp, a, scratch);
    if (threadIdx.x == 0) out[0] = t.mu, out[1] = t.sigma, out[2] = t.nu;
  } else {
    const double nu = estimate_nu<NT>(smp, a, b, scratch);
    if (threadIdx.x == 0) out[0] = nu;
  }
}
int launch_tdist_vec(const double* r, long long n, int mode, double a, double b, double* out,
                     cudaStream_t s) {
  cudaFuncSetAttribute(k_tdist_vec, cudaFuncAttributeMaxDynamicSharedMemorySize, kMaxSample * 8);
  KScope ks_("tdist_vec", s);
  k_tdist_vec<<<1, kTdistThreads, kMaxSample * 8, s>>>(r, n, mode, a, b, out);
  return 0;
}

// ---------------------------------------------------------------------------
// Self-test of div_rcp against IEEE division on n random operand pairs spanning
// the ranges the warp sees (numerators |a| < 2^20 incl. integers, divisors
// b in [1e-12, 1e6]).  Counts mismatches (bitwise).
__device__ __forceinline__ unsigned long long mix64(unsigned long long z) {
  z += 0x9e3779b97f4a7c15ull;
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}
__global__ void k_selftest_div(unsigned long long n, unsigned long long seed,
                               unsigned long long* mismatches) {
  unsigned long long bad = 0;
  for (unsigned long long i = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x; i < n;
       i += (unsigned long long)gridDim.x * blockDim.x) {
    const unsigned long long r1 = mix64(seed * 0x100000001ull + 2 * i), r2 = mix64(seed + 2 * i + 1);
    const double u1 = (r1 >> 11) * (1.0 / 9007199254740992.0);
    const double u2 = (r2 >> 11) * (1.0 / 9007199254740992.0);
    double a = (i & 3) == 0 ? (double)((r1 >> 40) % 2048) : (u1 - 0.5) * exp2(40.0 * u2 - 20.0);
    const double b = exp2(-39.9 + 59.8 * u2) * (1.0 + u1);
    const double r = __drcp_rn(b);
    const double q1 = div_rcp(a, b, r), q2 = a / b;
    if (__double_as_longlong(q1) != __double_as_longlong(q2)) ++bad;
    if (__double_as_longlong(r) != __double_as_longlong(1.0 / b)) ++bad;
  }
  if (bad) atomicAdd(mismatches, bad);
}

// FP64 FMA throughput probe: 8 independent DFMA chains per thread, all SMs.
__global__ void k_fp64_peak(int iters, double seed, double* out) {
  double a[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) a[i] = seed + threadIdx.x * 1e-9 + i;
  const double b = 0.999999999, c = 1e-12;
  for (int it = 0; it < iters; ++it)
#pragma unroll
    for (int i = 0; i < 8; ++i) a[i] = fma(a[i], b, c);
  double s = 0.0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += a[i];
  if (s == 42.0) out[0] = s;  // keep the chains alive
}

double measure_fp64_tflops(cudaStream_t s) {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  double* out;
  cudaMalloc(&out, sizeof(double));
  const int blocks = sms * 8, threads = 256, iters = 4096;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  k_fp64_peak<<<blocks, threads, 0, s>>>(64, 1.0, out);  // warm-up
  cudaEventRecord(e0, s);
  k_fp64_peak<<<blocks, threads, 0, s>>>(iters, 1.0, out);
  cudaEventRecord(e1, s);
  cudaEventSynchronize(e1);
  float ms = 0.f;
  cudaEventElapsedTime(&ms, e0, e1);
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaFree(out);
  const double flops = 2.0 * 8.0 * iters * (double)blocks * threads;
  return flops / (ms * 1e-3) / 1e12;
}

int selftest_division(unsigned long long n, unsigned long long seed, unsigned long long* out,
                      cudaStream_t s) {
  unsigned long long* d;
  if (cudaMalloc(&d, sizeof(*d)) != cudaSuccess) return 1;
  cudaMemsetAsync(d, 0, sizeof(*d), s);
  {
    KScope ks_("selftest_div", s);
    k_selftest_div<<<148 * 8, 256, 0, s>>>(n, seed, d);
  }
  cudaMemcpyAsync(out, d, sizeof(*d), cudaMemcpyDeviceToHost, s);
  cudaStreamSynchronize(s);
  cudaFree(d);
  return cudaGetLastError() == cudaSuccess ? 0 : 1;
}

}  // namespace rgbid_b200
