// Keyframe fusion, covisibility, depth correction, forward registration and the
// device-side synthetic pair generator (bench inputs).
//
//  k_integrate      integrate_frame — src/fusion.cpp:68-95; k frames fused per pixel
//                   (the per-pixel state depends only on the same pixel, so one
//                   launch over k frames is bit-identical to k sequential calls).
//  k_covisibility   count_visible — src/fusion.cpp:26-50 (both directions, exact
//                   integer counts via 64-bit atomics).
//  k_correct_depth  correct_inverse_depth + depth_poly — src/camera.cpp:54-81
//  k_rectify        inverse_warp with f_w = K distort(K^-1 p) — src/warping.cpp:8-18,
//                   src/camera.cpp:11-22,41-45 (distorted-sensor frames, config 4, k != 0)
//  k_undistort      undistort — src/camera.cpp:24-39 (per point, fixed-point iteration)
//  k_splat/k_gather forward_register — src/warping.cpp:20-74 (z-buffer splat via
//                   64-bit atomicMax on order-preserving keys: the max is
//                   independent of write order, as SPEC:316-317 requires)
#include <cuda_runtime.h>
#include <math_constants.h>

#include <cstdint>

#include "align_kernels.cuh"
#include "fusion_kernels.cuh"

namespace rgbid_b200 {

__device__ __forceinline__ bool fvalid(double v) { return isfinite(v); }

__device__ __forceinline__ double bilinear_f(const double* __restrict__ img, int w, int h, double x,
                                             double y) {
  if (!(x >= 0.0 && x <= w - 1.0 && y >= 0.0 && y <= h - 1.0)) return CUDART_NAN;
  const int x0 = (int)floor(x), y0 = (int)floor(y);
  const int x1 = min(x0 + 1, w - 1), y1 = min(y0 + 1, h - 1);
  const double fx = x - x0, fy = y - y0;
  const double v00 = __ldg(img + (size_t)y0 * w + x0), v10 = __ldg(img + (size_t)y0 * w + x1);
  const double v01 = __ldg(img + (size_t)y1 * w + x0), v11 = __ldg(img + (size_t)y1 * w + x1);
  if (!fvalid(v00) || !fvalid(v10) || !fvalid(v01) || !fvalid(v11)) return CUDART_NAN;
  return (1 - fy) * ((1 - fx) * v00 + fx * v10) + fy * ((1 - fx) * v01 + fx * v11);
}

// ---------------------------------------------------------------------------
// integrate_frame over k frames (frames in call order).
//
// Correctly rounded a / b from r = RN(1/b) (Markstein; bit-identical to IEEE a / b
// for normal operands, rgbid_selftest_division): the quotients sharing a divisor
// (p / w_kf, x_B / z) cost one reciprocal.  Divisors outside [1e-300, 1e300] take
// the IEEE division.
__device__ __forceinline__ double fdiv_rcp(double a, double b, double r) {
  const double q = a * r;
  const double e = fma(-b, q, a);
  return fma(e, r, q);
}
__device__ __forceinline__ bool rcp_safe(double b) {
  const double m = fabs(b);
  return m > 1e-300 && m < 1e300;
}

// one frame into one keyframe pixel (x, y): src/fusion.cpp:68-95 with W_A = the
// keyframe's current W (the per-pixel state depends only on this pixel).  Written
// branch-free (a validity predicate, safe operands, always-issued tap loads) so the
// chains of several pixels interleave; every test and expression is the
// reference's, in its order.
__device__ __forceinline__ void integrate_px(const FuseFrame& F, int x, int y, int w, int h,
                                             double gate, double& w_kf, double& c_kf) {
  const WarpMats& m = F.wm;
  // inverse_geometric_warp inverse depth at this pixel (src/warping.cpp:96-111)
  bool ok = fvalid(w_kf) && w_kf > 0.0;
  const double wa = ok ? w_kf : 1.0;
  double qx, qy, qz;
  if (rcp_safe(wa)) {
    qz = __drcp_rn(wa);
    qx = fdiv_rcp((double)x, wa, qz);
    qy = fdiv_rcp((double)y, wa, qz);
  } else {
    qx = x / wa;
    qy = y / wa;
    qz = 1.0 / wa;
  }
  const double xb0 = red3(m.Rt_BA[0] * qx, m.Rt_BA[1] * qy, m.Rt_BA[2] * qz) + m.tt_BA[0];
  const double xb1 = red3(m.Rt_BA[3] * qx, m.Rt_BA[4] * qy, m.Rt_BA[5] * qz) + m.tt_BA[1];
  const double xb2 = red3(m.Rt_BA[6] * qx, m.Rt_BA[7] * qy, m.Rt_BA[8] * qz) + m.tt_BA[2];
  ok = ok && xb2 > 1e-12;
  const double z = ok ? xb2 : 1.0;
  double bx, by;
  if (rcp_safe(z)) {
    const double r = __drcp_rn(z);
    bx = fdiv_rcp(xb0, z, r);
    by = fdiv_rcp(xb1, z, r);
  } else {
    bx = xb0 / z;
    by = xb1 / z;
  }
  // bilinear(frame.W, b) — inc/image.hpp:51-62
  const bool inb = ok && (bx >= 0.0 && bx <= w - 1.0 && by >= 0.0 && by <= h - 1.0);
  const double sx = inb ? bx : 0.0, sy = inb ? by : 0.0;
  const int x0 = (int)floor(sx), y0 = (int)floor(sy);
  const int dx = x0 + 1 < w ? 1 : 0, dy = y0 + 1 < h ? w : 0;
  const double fx = sx - x0, fy = sy - y0;
  const double* __restrict__ Wf = F.W;
  const int i00 = y0 * w + x0;
  const double v00 = __ldg(Wf + i00), v10 = __ldg(Wf + i00 + dx), v01 = __ldg(Wf + i00 + dy),
               v11 = __ldg(Wf + i00 + dy + dx);
  const double w_meas = (1 - fy) * ((1 - fx) * v00 + fx * v10) + fy * ((1 - fx) * v01 + fx * v11);
  ok = inb && fvalid(v00) && fvalid(v10) && fvalid(v01) && fvalid(v11) && fvalid(w_meas) &&
       w_meas > 0.0;
  const double rz = red3(m.Rt_AB[6] * bx, m.Rt_AB[7] * by, m.Rt_AB[8] * 1.0);
  const double za = rz / (ok ? w_meas : 1.0) + m.tt_AB[2];
  ok = ok && za > 1e-12;
  const double w_new = 1.0 / (ok ? za : 1.0);
  // fusion update — src/fusion.cpp:78-92 (w_b == w_meas: same bilinear call)
  ok = ok && fabs(w_new - w_kf) < gate;
  const double num = 1.0 - w_meas * m.tt_BA[2];
  const double den = red3(m.Rt_BA[6] * x, m.Rt_BA[7] * y, m.Rt_BA[8] * 1.0);
  const double t = num * num / den;
  const double c_k = t * t;
  ok = ok && isfinite(c_k) && c_k > 0.0;
  const double wn = (w_kf * c_kf + c_k * w_new) / (c_kf + c_k);
  if (ok) {
    w_kf = wn;
    c_kf = c_kf + c_k;
  }
}

// k frames, kIntPx pixels per thread (independent chains interleaved: the
// per-frame chain 1/w_kf -> x_B -> taps -> z_A -> update is serial per pixel), so
// that every keyframe pixel of a VGA frame is resident in one wave; the frames'
// warp matrices are staged in shared memory, kIntStage frames at a time.
constexpr int kIntPx = 2, kIntThreads = 256, kIntStage = 32;
__global__ void __launch_bounds__(kIntThreads) k_integrate(const FuseFrame* __restrict__ frames,
                                                           int k, double* __restrict__ kfW,
                                                           double* __restrict__ kfC, int w, int h,
                                                           double sigma_w) {
  __shared__ FuseFrame sf[kIntStage];
  const int n = w * h;
  const int base = blockIdx.x * (kIntThreads * kIntPx) + threadIdx.x;
  double wk[kIntPx], ck[kIntPx];
  int px[kIntPx], py[kIntPx];
#pragma unroll
  for (int j = 0; j < kIntPx; ++j) {
    const int i = base + j * kIntThreads;
    const bool in = i < n;
    wk[j] = in ? kfW[i] : CUDART_NAN;  // out-of-range pixels: holes, never updated
    ck[j] = in ? kfC[i] : 0.0;
    py[j] = in ? i / w : 0;
    px[j] = in ? i - py[j] * w : 0;
  }
  const double gate = 3.0 * sigma_w;
  for (int f0 = 0; f0 < k; f0 += kIntStage) {
    const int nf = min(kIntStage, k - f0);
    __syncthreads();
    for (int t = threadIdx.x; t < nf * (int)(sizeof(FuseFrame) / 8); t += kIntThreads)
      reinterpret_cast<double*>(sf)[t] = reinterpret_cast<const double*>(frames + f0)[t];
    __syncthreads();
    for (int f = 0; f < nf; ++f) {
#pragma unroll
      for (int j = 0; j < kIntPx; ++j) integrate_px(sf[f], px[j], py[j], w, h, gate, wk[j], ck[j]);
    }
  }
#pragma unroll
  for (int j = 0; j < kIntPx; ++j) {
    const int i = base + j * kIntThreads;
    if (i < n) {
      kfW[i] = wk[j];
      kfC[i] = ck[j];
    }
  }
}

void launch_integrate(const FuseFrame* frames_dev, int k, double* kfW, double* kfC, int w, int h,
                      double sigma_w, cudaStream_t s) {
  KScope ks_("integrate", s);
  const int per = kIntThreads * kIntPx;
  k_integrate<<<(w * h + per - 1) / per, kIntThreads, 0, s>>>(frames_dev, k, kfW, kfC, w, h,
                                                              sigma_w);
}

// ---------------------------------------------------------------------------
// count_visible for both directions (blockIdx.y = direction)
__global__ void __launch_bounds__(256) k_covisibility(CovisDir d0, CovisDir d1, int w, int h,
                                                      double gate,
                                                      unsigned long long* __restrict__ counts) {
  const CovisDir& D = blockIdx.y ? d1 : d0;
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  int valid = 0, visible = 0;
  if (i < w * h) {
    const int y = i / w, x = i - y * w;
    const double w_a = __ldg(D.WA + i);
    if (fvalid(w_a) && w_a > 0.0) {
      valid = 1;
      const double qx = x / w_a, qy = y / w_a, qz = 1.0 / w_a;
      const double xb0 = red3(D.Rt[0] * qx, D.Rt[1] * qy, D.Rt[2] * qz) + D.tt[0];
      const double xb1 = red3(D.Rt[3] * qx, D.Rt[4] * qy, D.Rt[5] * qz) + D.tt[1];
      const double xb2 = red3(D.Rt[6] * qx, D.Rt[7] * qy, D.Rt[8] * qz) + D.tt[2];
      if (xb2 > 1e-12) {
        const double w_b = 1.0 / xb2;
        const double px = xb0 / xb2, py = xb1 / xb2;
        if (px >= 0.0 && px <= w - 1.0 && py >= 0.0 && py <= h - 1.0) {
          const double w_meas = bilinear_f(D.WB, w, h, px, py);
          if (fvalid(w_meas) && fabs(w_meas - w_b) < gate) visible = 1;
        }
      }
    }
  }
  // exact integer block reduction, then one 64-bit atomic per block
  __shared__ int sv[8], ss[8];
  int v = valid, s = visible;
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
    v += __shfl_down_sync(0xffffffffu, v, off);
    s += __shfl_down_sync(0xffffffffu, s, off);
  }
  if ((threadIdx.x & 31) == 0) {
    sv[threadIdx.x >> 5] = v;
    ss[threadIdx.x >> 5] = s;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    long long tv = 0, ts = 0;
    for (int k = 0; k < 8; ++k) {
      tv += sv[k];
      ts += ss[k];
    }
    atomicAdd(&counts[2 * blockIdx.y + 0], (unsigned long long)tv);
    atomicAdd(&counts[2 * blockIdx.y + 1], (unsigned long long)ts);
  }
}

void launch_covisibility(const CovisDir& d0, const CovisDir& d1, int w, int h, double sigma_w,
                         unsigned long long* counts_dev, cudaStream_t s) {
  cudaMemsetAsync(counts_dev, 0, 4 * sizeof(unsigned long long), s);
  KScope ks_("covisibility", s);
  k_covisibility<<<dim3((w * h + 255) / 256, 2), 256, 0, s>>>(d0, d1, w, h, 3.0 * sigma_w,
                                                              counts_dev);
}

// ---------------------------------------------------------------------------
// Brown distortion of a normalized point — src/camera.cpp:11-22, expression order
// as written (z is not needed by any caller)
__device__ __forceinline__ void distort_d(const rgbid_intrinsics& K, double x, double y, double& ox,
                                          double& oy) {
  const double r2 = x * x + y * y;
  const double r4 = r2 * r2;
  const double r6 = r4 * r2;
  const double radial = K.k[0] * r2 + K.k[1] * r4 + K.k[4] * r6;
  ox = (1.0 + radial) * x;
  oy = (1.0 + radial) * y;
  ox += 2.0 * K.k[2] * x * y + K.k[3] * (r2 + 2.0 * x * x);
  oy += 2.0 * K.k[3] * x * y + K.k[2] * (r2 + 2.0 * y * y);
}

// rectification of a distorted-sensor image pair (I and W of one frame, blockIdx.y):
// out(p) = bilinear(src, f_w(p)), f_w(p) = project(K, ((x - cx) / fx, (y - cy) / fy, 1))
__global__ void k_rectify(const double* __restrict__ I, const double* __restrict__ W, int w, int h,
                          rgbid_intrinsics K, double* __restrict__ oI, double* __restrict__ oW) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= w * h) return;
  const int y = i / w, x = i - y * w;
  const double mx = (x - K.cx) / K.fx, my = (y - K.cy) / K.fy;
  double dx, dy;
  distort_d(K, mx, my, dx, dy);
  const double qx = K.fx * dx + K.cx, qy = K.fy * dy + K.cy;
  const double* src = blockIdx.y ? W : I;
  double* out = blockIdx.y ? oW : oI;
  out[i] = bilinear_f(src, w, h, qx, qy);
}

void launch_rectify(const double* I, const double* W, int w, int h, const rgbid_intrinsics& K,
                    double* oI, double* oW, cudaStream_t s) {
  KScope ks_("rectify", s);
  // one grid row per map; W == nullptr: I only
  k_rectify<<<dim3((w * h + 255) / 256, W ? 2 : 1), 256, 0, s>>>(I, W, w, h, K, oI, oW);
}

// undistort — src/camera.cpp:24-39: fixed-point iteration m_u -= distort(m_u) - m_d,
// at most 50 steps, |err|_inf < 1e-10; ok = 0 is the reference's std::nullopt
__global__ void k_undistort(const double* __restrict__ md, long long n, rgbid_intrinsics K,
                            double* __restrict__ mu, uint8_t* __restrict__ ok) {
  const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double tx = md[2 * i], ty = md[2 * i + 1];
  bool dist = false;
  for (int k = 0; k < 5; ++k) dist |= K.k[k] != 0.0;  // Intrinsics::has_distortion
  double ux = tx, uy = ty;
  uint8_t good = 0;
  if (!dist) {
    good = 1;
  } else {
    for (int it = 0; it < 50 && !good; ++it) {
      double dx, dy;
      distort_d(K, ux, uy, dx, dy);
      const double ex = dx - tx, ey = dy - ty;
      ux -= ex;
      uy -= ey;
      if (dmax_std(fabs(ex), fabs(ey)) < 1e-10) good = 1;
    }
    if (!good) {
      double dx, dy;
      distort_d(K, ux, uy, dx, dy);
      if (dmax_std(fabs(dx - tx), fabs(dy - ty)) < 1e-10) good = 1;
    }
  }
  ok[i] = good;
  mu[2 * i] = good ? ux : 0.0;
  mu[2 * i + 1] = good ? uy : 0.0;
}

void launch_undistort(const double* md, long long n, const rgbid_intrinsics& K, double* mu,
                      uint8_t* ok, cudaStream_t s) {
  KScope ks_("undistort", s);
  k_undistort<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(md, n, K, mu, ok);
}

// ---------------------------------------------------------------------------
// correct_inverse_depth — src/camera.cpp:54-81
__device__ __forceinline__ double depth_poly_d(const double* q, double cx, double cy, double fx,
                                               double fy, double px, double py) {
  const double mx = (px - cx) / fx;
  const double my = (py - cy) / fy;
  const double r2 = mx * mx + my * my;
  return q[0] + q[1] * r2 + q[2] * r2 * r2 + q[3] * r2 * r2 * r2 + q[4] * mx + q[5] * my +
         q[6] * mx * my + q[7] * mx * mx * my + q[8] * mx * my * my;
}

__global__ void k_correct_depth(const double* __restrict__ Wm, int w, int h,
                                rgbid_depth_intrinsics d, double fx, double fy, double cx,
                                double cy, int spatial, double* __restrict__ out) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= w * h) return;
  const int y = i / w, x = i - y * w;
  const int sx = (int)lround(x - d.p0[0]);
  const int sy = (int)lround(y - d.p0[1]);
  double o = CUDART_NAN;
  if (sx >= 0 && sx < w && sy >= 0 && sy < h) {
    const double w_m = Wm[(size_t)sy * w + sx];
    if (fvalid(w_m)) {
      double v = d.beta1 * w_m + d.beta0;
      if (spatial)
        v = depth_poly_d(d.q1, cx, cy, fx, fy, x, y) * v + depth_poly_d(d.q0, cx, cy, fx, fy, x, y);
      o = v;
    }
  }
  out[i] = o;
}

void launch_correct_depth(const double* Wm, int w, int h, const rgbid_depth_intrinsics& d,
                          const rgbid_intrinsics& K, int spatial, double* out, cudaStream_t s) {
  KScope ks_("correct_depth", s);
  k_correct_depth<<<(w * h + 255) / 256, 256, 0, s>>>(Wm, w, h, d, K.fx, K.fy, K.cx, K.cy, spatial,
                                                      out);
}

// ---------------------------------------------------------------------------
// forward_register — src/warping.cpp:20-74
__device__ __forceinline__ unsigned long long order_key(double v) {
  const long long b = __double_as_longlong(v);
  return b >= 0 ? ((unsigned long long)b | 0x8000000000000000ull) : ~(unsigned long long)b;
}
__device__ __forceinline__ double key_value(unsigned long long k) {
  if (k == 0ull) return CUDART_NAN;  // empty slot (hole)
  const unsigned long long b = (k & 0x8000000000000000ull) ? (k & 0x7fffffffffffffffull) : ~k;
  return __longlong_as_double((long long)b);
}

__global__ void k_splat(const double* __restrict__ WA, int w, int h, RegisterMats r,
                        unsigned long long* __restrict__ inter, int iw, int ih) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= w * h) return;
  const int y = i / w, x = i - y * w;
  const double wv = WA[i];
  if (!fvalid(wv)) return;
  const double denom = 1.0 - wv * r.tt[2];
  if (denom <= 1e-12) return;
  const double w_bt = wv / denom;
  const double pbx = (x - wv * r.tt[0]) / denom;
  const double pby = (y - wv * r.tt[1]) / denom;
  const double half = 0.5 * (w_bt / wv);
  const int x0 = (int)lround(pbx - half), x1 = (int)lround(pbx + half);
  const int y0 = (int)lround(pby - half), y1 = (int)lround(pby + half);
  const unsigned long long key = order_key(w_bt);
  for (int ty = max(y0, 0); ty <= y1 && ty < ih; ++ty)
    for (int tx = max(x0, 0); tx <= x1 && tx < iw; ++tx)
      atomicMax(&inter[(size_t)ty * iw + tx], key);
}

__global__ void k_gather_register(const unsigned long long* __restrict__ inter, int iw, int ih,
                                  RegisterMats r, int wb, int hb, double* __restrict__ out) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= wb * hb) return;
  const int y = i / wb, x = i - y * wb;
  double o = CUDART_NAN;
  const double rx = red3(r.Rt_AB[0] * x, r.Rt_AB[1] * y, r.Rt_AB[2] * 1.0);
  const double ry = red3(r.Rt_AB[3] * x, r.Rt_AB[4] * y, r.Rt_AB[5] * 1.0);
  const double rz = red3(r.Rt_AB[6] * x, r.Rt_AB[7] * y, r.Rt_AB[8] * 1.0);
  if (rz > 1e-12) {
    const double bx = rx / rz, by = ry / rz;
    const int xi = (int)lround(bx), yi = (int)lround(by);
    if (xi >= 0 && xi < iw && yi >= 0 && yi < ih) {
      const double wbt = key_value(inter[(size_t)yi * iw + xi]);
      if (fvalid(wbt)) o = wbt * rz;
    }
  }
  out[i] = o;
}

void launch_forward_register(const double* WA, int w, int h, const RegisterMats& r,
                             unsigned long long* inter, int iw, int ih, int wb, int hb,
                             double* out, cudaStream_t s) {
  cudaMemsetAsync(inter, 0, sizeof(unsigned long long) * (size_t)iw * ih, s);
  {
    KScope ks_("register_splat", s);
    k_splat<<<(w * h + 255) / 256, 256, 0, s>>>(WA, w, h, r, inter, iw, ih);
  }
  KScope ks_("register_gather", s);
  k_gather_register<<<(wb * hb + 255) / 256, 256, 0, s>>>(inter, iw, ih, r, wb, hb, out);
}

// ---------------------------------------------------------------------------
// Device synthetic pair (bench inputs, synth_scene.cuh): render_plane of
// tests/synthetic.hpp:24-50 with plane_texture at tex_scale * (X, Y), optional
// Gaussian noise (counter-based hash + Box-Muller), a 20% near occluder
// (test_alignment.cpp:220-232) and seeded holes / a border band.
__device__ __forceinline__ double plane_texture_d(double x, double y) {
  return 0.5 + 0.2 * sin(7.3 * x) * cos(5.9 * y) + 0.15 * sin(3.1 * x + 2.7 * y) +
         0.1 * cos(11.0 * x - 4.0 * y);
}
__device__ __forceinline__ double gauss(unsigned long long key) {
  const unsigned long long a = synth_splitmix(key), b = synth_splitmix(key ^ 0xda3e39cb94b95bdbull);
  const double u1 = ((a >> 11) + 0.5) * (1.0 / 9007199254740992.0);
  const double u2 = ((b >> 11) + 0.5) * (1.0 / 9007199254740992.0);
  return sqrt(-2.0 * log(u1)) * cos(6.283185307179586 * u2);
}

__global__ void k_render(SynthView v, double* __restrict__ I, double* __restrict__ W) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= v.w * v.h) return;
  const int y = i / v.w, x = i - y * v.w;
  const V3 p = {{(double)x, (double)y, 1.0}};
  const V3 kp = m3_mulv(v.Kinv, p);
  const V3 r = m3_mulv(v.R, kp);
  const double denom = red3(v.n[0] * r.v[0], v.n[1] * r.v[1], v.n[2] * r.v[2]);
  double iv = CUDART_NAN, wv = CUDART_NAN;
  if (fabs(denom) >= 1e-12) {
    const double lambda = -(red3(v.n[0] * v.t[0], v.n[1] * v.t[1], v.n[2] * v.t[2]) + v.d) / denom;
    if (lambda > 0.05) {
      const double X = v.t[0] + lambda * r.v[0], Y = v.t[1] + lambda * r.v[1];
      iv = plane_texture_d(v.tex_scale * X, v.tex_scale * Y);
      wv = 1.0 / lambda;
    }
  }
  if (v.noise_i > 0.0 && fvalid(iv)) iv += v.noise_i * gauss(v.seed * 0x100000000ull + 2ull * i);
  if (v.noise_w > 0.0 && fvalid(wv)) wv += v.noise_w * gauss(v.seed * 0x100000000ull + 2ull * i + 1);
  if (v.occluder && x < v.w / 5) {
    iv = plane_texture_d(7.0 + 0.1 * x * 80.0 / v.w, 3.0 + 0.1 * y * 80.0 / v.w);
    wv = 1.0;
  }
  if (synth_hole_i(v, i)) iv = CUDART_NAN;
  if (synth_hole_w(v, i, x, y)) wv = CUDART_NAN;
  I[i] = iv;
  W[i] = wv;
}

void launch_render(const SynthView& v, double* I, double* W, cudaStream_t s) {
  KScope ks_("synth_render", s);
  k_render<<<(v.w * v.h + 255) / 256, 256, 0, s>>>(v, I, W);
}

// ---------------------------------------------------------------------------
// Frame ingest — load_frame's pixel decode (src/dataset.cpp:97-116): BGR8 ->
// gray = (0.299 R + 0.587 G + 0.114 B) / 255, depth16 -> scale / raw (0 = hole).
__global__ void k_decode_frame(const uint8_t* __restrict__ bgr, const uint16_t* __restrict__ depth,
                               int n, double scale, double* __restrict__ I,
                               double* __restrict__ W) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  if (bgr) {
    const double b = bgr[3 * i], g = bgr[3 * i + 1], r = bgr[3 * i + 2];
    I[i] = (0.299 * r + 0.587 * g + 0.114 * b) / 255.0;
  }
  const uint16_t raw = depth[i];
  W[i] = raw == 0 ? CUDART_NAN : scale / (double)raw;
}

void launch_decode_frame(const uint8_t* bgr, const uint16_t* depth, int n, double scale, double* I,
                         double* W, cudaStream_t s) {
  KScope ks_("decode_frame", s);
  k_decode_frame<<<(n + 255) / 256, 256, 0, s>>>(bgr, depth, n, scale, I, W);
}

}  // namespace rgbid_b200
